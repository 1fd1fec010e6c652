// f64_emu.cu — MM_F64_EMU: the binary64 product C = A·B (the paper's `double`
// precision) computed on the INT8 tensor cores by exact digit slicing (the Ozaki
// scheme), for problems where the 2.25 / 4.5 PFLOP/s tensor pipes beat the 37 TFLOP/s DMMA pipe.
//
//   * Row i of A is scaled by 2^-e_i (|a_ik| < 2^e_i, e_i the frexp exponent of the row maximum)
//     and each scaled element x ∈ (-1, 1) is cut into S = 8 signed 7-bit digits
//     x = Σ_u d_u 2^(-7u), d_u = trunc(128 · remainder) ∈ [-127, 127] — exact in binary64 (a
//     multiplication by 2^7 and the subtraction of an integer part are exact), 56 bits ≥ 53.
//     Column j of B likewise with 2^-f_j into digits g_v.
//   * a_ik·b_kj summed over k = Σ_{u,v} 2^(e_i + f_j - 7(u+v)) Σ_k d_u,ik g_v,kj; each inner sum is
//     an INT8 product with INT32 accumulation, exact while (#pairs)·n·127² < 2^31 (n ≤ 33288 for 4
//     pairs — C5's n = 32768 fits 4).  Pairs of equal weight w = u+v are one INT8 GEMM whose K
//     runs over the pairs: A digits stored [row][u][k], B digits [8-v][k][col], so the pairs of a
//     weight are contiguous K ranges of both (no copy).  Pairs with w ≤ S+1 (36 of 64) are kept; the
//     dropped ones weigh ≤ 2^(-70) relative to the row/column scales.
//   * Each weight's INT32 result is scaled by the exact power of two and added into C in binary64,
//     smallest weights first (fixed order: run-to-run identical).
// Accuracy: exact integer inputs (|x| < 2^14) give exact results (bit-identical to the oracle);
// U[-1,1) inputs give normalised errors ~1e-16, like DMMA (tests/test_gpu_parity.py).
#include <climits>
#include <cstdint>

#include "ctx.h"
#include "kernels.h"

namespace mmb {

namespace {

constexpr int kDigits = 8;           // S: 8 x 7 bits = 56 >= 53
constexpr int kExpBias = 4096;       // encoded exponent (0 = all-zero row / column)
constexpr int64_t kMaxPairs = 8;     // INT8 products summed in one INT32 accumulator (n permitting)

__device__ __forceinline__ int dec_exp(int v) { return v ? v - kExpBias : 0; }

// e[i] = bias + frexp exponent of max_k |A[i][k]| (0 if the row is zero)
__global__ void row_exp_kernel(const double* __restrict__ A, int64_t lda, int64_t n, int* __restrict__ e) {
  const int64_t i = blockIdx.x;
  double mx = 0.0;
  for (int64_t k = threadIdx.x; k < n; k += blockDim.x) mx = fmax(mx, fabs(A[i * lda + k]));
  __shared__ double red[32];
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x < 32) {
    mx = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (threadIdx.x == 0) {
      int ex = 0;
      if (mx > 0.0) frexp(mx, &ex);
      e[i] = mx > 0.0 ? ex + kExpBias : 0;
    }
  }
}

// f[j] = max over rows (atomicMax of the encoded exponent; f zeroed before)
__global__ void col_exp_kernel(const double* __restrict__ B, int64_t ldb, int64_t n, int64_t p, int64_t rows_per,
                               int* __restrict__ f) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(n, r0 + rows_per);
  double mx = 0.0;
  for (int64_t k = r0; k < r1; ++k) mx = fmax(mx, fabs(B[k * ldb + j]));
  if (mx > 0.0) {
    int ex = 0;
    frexp(mx, &ex);
    atomicMax(f + j, ex + kExpBias);
  }
}

// 8 digits of x ∈ (-1, 1): d_u = trunc(128 r_{u-1}), r_u = 128 r_{u-1} - d_u (exact)
__device__ __forceinline__ void digits(double x, int (&d)[kDigits]) {
#pragma unroll
  for (int u = 0; u < kDigits; ++u) {
    x *= 128.0;
    const double t = trunc(x);
    d[u] = (int)t;
    x -= t;
  }
}

// A digits: Ad[(i*8 + u)*kp + k] (k >= n zero); 4 consecutive k per thread, packed 32-bit stores
__global__ void slice_a_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t n, int64_t kp,
                               const int* __restrict__ e, int8_t* __restrict__ Ad) {
  const int64_t q4 = kp / 4;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * q4; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / q4, k0 = (t % q4) * 4;
    const int sc = -dec_exp(e[i]);
    uint32_t w[kDigits] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t k = k0 + c;
      int d[kDigits];
      digits(k < n ? ldexp(A[i * lda + k], sc) : 0.0, d);
#pragma unroll
      for (int u = 0; u < kDigits; ++u) w[u] |= ((uint32_t)(uint8_t)(int8_t)d[u]) << (8 * c);
    }
#pragma unroll
    for (int u = 0; u < kDigits; ++u) *reinterpret_cast<uint32_t*>(Ad + (i * kDigits + u) * kp + k0) = w[u];
  }
}

// B digits: Bd[((8-v)*kp + k)*p + j] for digit v = 1..8 (plane 0 holds digit 8); k >= n rows zero.
// P4: p % 4 == 0 -> 4 consecutive columns per thread, packed 32-bit stores.
template <bool P4>
__global__ void slice_b_kernel(const double* __restrict__ B, int64_t ldb, int64_t n, int64_t p, int64_t kp,
                               const int* __restrict__ f, int8_t* __restrict__ Bd) {
  const int64_t cw = P4 ? p / 4 : p;
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < kp * cw; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = t / cw, j0 = (t % cw) * (P4 ? 4 : 1);
    if constexpr (P4) {
      uint32_t w[kDigits] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        int d[kDigits];
        digits(k < n ? ldexp(B[k * ldb + j0 + c], -dec_exp(f[j0 + c])) : 0.0, d);
#pragma unroll
        for (int u = 0; u < kDigits; ++u) w[u] |= ((uint32_t)(uint8_t)(int8_t)d[u]) << (8 * c);
      }
#pragma unroll
      for (int u = 0; u < kDigits; ++u)  // digit v = u + 1 -> plane 8 - v = 7 - u
        *reinterpret_cast<uint32_t*>(Bd + ((int64_t)(kDigits - 1 - u) * kp + k) * p + j0) = w[u];
    } else {
      int d[kDigits];
      digits(k < n ? ldexp(B[k * ldb + j0], -dec_exp(f[j0])) : 0.0, d);
#pragma unroll
      for (int u = 0; u < kDigits; ++u) Bd[((int64_t)(kDigits - 1 - u) * kp + k) * p + j0] = (int8_t)d[u];
    }
  }
}

// C (+)= S · 2^(e_i + f_j - 7w); `assign` overwrites (the first weight of a beta = 0 product)
__global__ void scale_acc_kernel(const int32_t* __restrict__ S, int64_t m, int64_t p, double* __restrict__ C,
                                 int64_t ldc, const int* __restrict__ e, const int* __restrict__ f, int w, int assign) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < m * p; t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = t / p, j = t % p;
    const double v = ldexp((double)S[t], dec_exp(e[i]) + dec_exp(f[j]) - 7 * w);
    double* c = C + i * ldc + j;
    *c = assign ? v : *c + v;
  }
}

inline int grid_for(int64_t work, int num_sms) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 16));
}

}  // namespace

int64_t f64_emu_kp(int64_t n) { return (n + 15) / 16 * 16; }

size_t f64_emu_scratch(int64_t m, int64_t n, int64_t p) {
  const int64_t kp = f64_emu_kp(n);
  return (size_t)(m * kDigits * kp) + (size_t)(kDigits * kp * p) + (size_t)(m * p * 4) + (size_t)((m + p) * 4) + 4 * 256;
}

mm_status gemm_f64_emu(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double* C, int64_t ldc, int beta_one, cudaStream_t s) {
  const int64_t kp = f64_emu_kp(n);
  const int64_t lim = (int64_t)INT32_MAX / (int64_t)(127 * 127);  // n x pairs bound for exact INT32 sums
  if (kp > lim) return set_err(ctx, MM_ERR_UNSUPPORTED, "MM_F64_EMU: n = %lld exceeds the exact-INT32 bound %lld", (long long)n, (long long)lim);
  const int64_t max_pairs = std::min<int64_t>(kMaxPairs, lim / kp);
  const size_t bA = (size_t)(m * kDigits * kp), bB = (size_t)(kDigits * kp * p), bS = (size_t)(m * p * 4);
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  const size_t need = up(bA) + up(bB) + up(bS) + up((size_t)m * 4) + up((size_t)p * 4);
  mm_status st = ensure_buffer(ctx, &ctx->emu_buf, &ctx->emu_bytes, need);
  if (st != MM_OK) return st;
  uint8_t* base = static_cast<uint8_t*>(ctx->emu_buf);
  int8_t* Ad = reinterpret_cast<int8_t*>(base);
  int8_t* Bd = reinterpret_cast<int8_t*>(base + up(bA));
  int32_t* S = reinterpret_cast<int32_t*>(base + up(bA) + up(bB));
  int* e = reinterpret_cast<int*>(base + up(bA) + up(bB) + up(bS));
  int* f = reinterpret_cast<int*>(base + up(bA) + up(bB) + up(bS) + up((size_t)m * 4));
  const int sms = ctx->num_sms;
  auto chk = [&](const char* what) -> mm_status {
    const cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "MM_F64_EMU %s launch failed: %s", what, cudaGetErrorString(ce));
    ++ctx->launches;
    return MM_OK;
  };
  // scales and digits
  row_exp_kernel<<<(unsigned)m, 256, 0, s>>>(A, lda, n, e);
  if ((st = chk("row exponents")) != MM_OK) return st;
  if (cudaMemsetAsync(f, 0, (size_t)p * 4, s) != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "MM_F64_EMU memset failed");
  const int64_t rows_per = std::max<int64_t>(64, (n + 63) / 64);
  col_exp_kernel<<<dim3((unsigned)((p + 255) / 256), (unsigned)((n + rows_per - 1) / rows_per)), 256, 0, s>>>(B, ldb, n, p,
                                                                                                           rows_per, f);
  if ((st = chk("column exponents")) != MM_OK) return st;
  slice_a_kernel<<<grid_for(m * (kp / 4), sms), 256, 0, s>>>(A, lda, m, n, kp, e, Ad);
  if ((st = chk("A digits")) != MM_OK) return st;
  if (p % 4 == 0) slice_b_kernel<true><<<grid_for(kp * (p / 4), sms), 256, 0, s>>>(B, ldb, n, p, kp, f, Bd);
  else slice_b_kernel<false><<<grid_for(kp * p, sms), 256, 0, s>>>(B, ldb, n, p, kp, f, Bd);
  if ((st = chk("B digits")) != MM_OK) return st;
  // weights w = u + v from the smallest (w = S + 1) to the largest (w = 2); each weight's pairs
  // u = u0..u1 (v = w - u) in chunks of at most max_pairs: one INT8 GEMM over K = chunk x kp
  bool first = true;
  for (int w = kDigits + 1; w >= 2; --w) {
    const int u0 = std::max(1, w - kDigits), u1 = std::min(kDigits, w - 1);
    for (int ua = u0; ua <= u1; ua += (int)max_pairs) {
      const int cnt = std::min<int>((int)max_pairs, u1 - ua + 1);
      const int q0 = kDigits - w + ua;  // B plane of digit v = w - ua
      const int8_t* Aw = Ad + (int64_t)(ua - 1) * kp;
      const int8_t* Bw = Bd + (int64_t)q0 * kp * p;
      st = gemm_ld(ctx, m, cnt * kp, p, MM_S8_S32, Aw, kDigits * kp, Bw, p, S, p, 0, s);
      if (st != MM_OK) return st;
      scale_acc_kernel<<<grid_for(m * p, sms), 256, 0, s>>>(S, m, p, C, ldc, e, f, w, (first && !beta_one) ? 1 : 0);
      if ((st = chk("scale-accumulate")) != MM_OK) return st;
      first = false;
    }
  }
  return MM_OK;
}

}  // namespace mmb
