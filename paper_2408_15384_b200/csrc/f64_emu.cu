// f64_emu.cu — MM_F64_EMU: the binary64 product C = A·B (the paper's `double`
// precision) computed on the INT8 tensor cores by exact modular arithmetic (the
// Ozaki scheme, second kind: integer scaling + Chinese remaindering), for problems where the
// 4.5 POPS INT8 pipe beats the 37 TFLOP/s DMMA pipe.
//
//   * Integer scaling.  Row i of A is scaled by 2^(β - e_i) (e_i = frexp exponent of the row
//     maximum, so |·| < 2^β) and rounded: a'_ik = rint(a_ik · 2^(β-e_i)), an exact binary64
//     integer with |a'| ≤ 2^β; column j of B likewise with 2^(β-f_j) into b'_kj.  The rounding
//     error is ≤ 2^-β of the row / column maximum (β ≥ 53: the binary64 rounding of that maximum);
//     an integer input stays an integer after the scaling (2^(β-e) ≥ 1), so it is not rounded.
//   * Residues.  N pairwise-coprime moduli m_1..m_N ≤ 256 (M = Π m_l); the symmetric residues
//     a'_ik mod m_l, b'_kj mod m_l lie in [-128, 127], so each C'_l = A'_l · B'_l is one INT8
//     product with INT32 accumulation, exact while n · 2^14 < 2^31 (n < 131072); all N run as one
//     batched launch (planes stacked along M) whose epilogue stores C'_l mod m_l as bytes
//     (gemm_tc.cu, GemmArgs::res_m / bat_rows).
//   * Reconstruction.  C' = A'·B' is an integer with |C'| ≤ n · 2^(2β); N and β are chosen so that
//     n · 2^(2β) ≤ M/2 - 1 with β ≥ 53 (N = 14..16 for n < 131072).  Garner's algorithm turns the
//     residues c_l = C'_l mod m_l into symmetric mixed-radix digits v_l (exact small-integer
//     arithmetic), C' = v_1 + m_1 (v_2 + m_2 (v_3 + ...)), evaluated by Horner's rule over digit
//     triples, plain binary64 while exact, then double-double (~2^-104 relative), rounded once to binary64 and scaled
//     by 2^-(2β - e_i - f_j) (exact unless the result is subnormal).
// Accuracy: exact integer inputs give exact results (bit-identical to the oracle); U[-1,1) inputs
// give normalised errors ~1e-17..1e-16, the accuracy class of DMMA (tests/test_gpu_parity.py).
// Inputs must be finite: an Inf or NaN is detected by the scale kernels and reported by
// mm_sync_check (C is then undefined; IEEE propagation needs MM_F64).
// Cost: N INT8 products (16 at C5) + O(N·(mn + np) + N²·mp) integer work in the residue and
// reconstruction kernels; DESIGN.md §6 K5 has the measured breakdown.
#include <climits>
#include <cmath>
#include <cstdint>

#include "ctx.h"
#include "kernels.h"
#include "knobs.h"

namespace mmb {

namespace {

constexpr int kMaxMod = 16;   // moduli used at most (n < 131072 needs at most 16 for β ≥ 53)
constexpr int kMinMod = 14;   // fewest moduli that give β ≥ 53 at n = 1
constexpr int kMinBeta = 53;  // bits kept of every row / column maximum
constexpr int kMaxBeta = 60;
constexpr int kExpBias = 4096;  // encoded exponent (0 = all-zero row / column)
// pairwise coprime, largest first (256 = 2^8, 255 = 3·5·17, 253 = 11·23, 247 = 13·19, 217 = 7·31,
// the rest prime)
constexpr int kMods[kMaxMod] = {256, 255, 253, 251, 247, 241, 239, 233, 229, 227, 223, 217, 211, 199, 197, 193};

// Garner tables, passed by value (kernel parameter space: constant-bank operands)
struct CrtTab {
  int nmod;                       // N
  int beta;                       // β
  int m[kMaxMod];                 // m_l
  // 0-based digits: C' = Σ_q v_q P_q with P_0 = 1, P_q = m[0] ... m[q-1]
  int pmod[kMaxMod][kMaxMod];     // pmod[q][k] = P_q · (P_k)^-1 mod m[k] for q < k
  int pinv[kMaxMod];              // (P_k mod m[k])^-1 mod m[k]
};

int inv_mod(int a, int m) {  // a^-1 mod m (gcd(a, m) = 1)
  int t = 0, nt = 1, r = m, nr = ((a % m) + m) % m;
  while (nr) {
    const int q = r / nr;
    int x = t - q * nt; t = nt; nt = x;
    x = r - q * nr; r = nr; nr = x;
  }
  return ((t % m) + m) % m;
}

// N and β for inner dimension n: the fewest moduli with β = floor((log2 M - 1 - log2 n) / 2) ≥ 53
bool crt_plan(int64_t n, int* nmod, int* beta) {
  double lm = 0.0;
  for (int l = 0; l < kMaxMod; ++l) {
    lm += std::log2((double)kMods[l]);
    if (l + 1 < kMinMod) continue;
    const double room = lm - 1.0 - std::log2((double)n) - 1e-9;
    const int b = (int)std::floor(room / 2.0);
    if (b >= kMinBeta) {
      *nmod = l + 1;
      *beta = std::min(b, kMaxBeta);
      return true;
    }
  }
  return false;
}

CrtTab make_tab(int nmod, int beta) {
  CrtTab t{};
  t.nmod = nmod;
  t.beta = beta;
  for (int l = 0; l < kMaxMod; ++l) {
    t.m[l] = kMods[l];
  }
  for (int k = 0; k < kMaxMod; ++k) {
    int pk = 1 % kMods[k];  // P_0 mod m[k]
    int pj[kMaxMod];
    for (int j = 0; j < k; ++j) {
      pj[j] = pk;  // P_j mod m[k]
      pk = (int)((int64_t)pk * kMods[j] % kMods[k]);
    }
    t.pinv[k] = k == 0 ? 1 : inv_mod(pk, kMods[k]);  // pk = P_k mod m[k]
    for (int j = 0; j < k; ++j) t.pmod[j][k] = (int)((int64_t)pj[j] * t.pinv[k] % kMods[k]);
  }
  return t;
}

__device__ __forceinline__ int dec_exp(int v) { return v ? v - kExpBias : 0; }

// 2^k for -1022 <= k <= 1023
__device__ __forceinline__ double pow2(int k) { return __longlong_as_double((long long)(k + 1023) << 52); }

// x·2^k, |k| ≤ 2044, in two exact steps of about k/2 (an element that underflows in the first step
// is below 2^-590 of its row / column maximum and rounds to 0 anyway)
__device__ __forceinline__ double scale2(double x, int k) {
  const int a = k / 2;
  return x * pow2(a) * pow2(k - a);
}

// x·2^k, |k| ≤ 3066, in three steps of about k/3: no intermediate underflows or overflows unless the
// result does (|x| ≥ 1 or 0), so the result is x·2^k rounded once
__device__ __forceinline__ double scale3(double x, int k) {
  const int a = k / 3, b = (k - a) / 2;
  return x * pow2(a) * pow2(b) * pow2(k - a - b);
}


// the moduli as compile-time constants once a loop over l is unrolled (x % m becomes a
// multiply-high, not a division)
__host__ __device__ constexpr int mod_at(int l) {
  return l == 0 ? 256 : l == 1 ? 255 : l == 2 ? 253 : l == 3 ? 251 : l == 4 ? 247 : l == 5 ? 241 : l == 6 ? 239
       : l == 7 ? 233 : l == 8 ? 229 : l == 9 ? 227 : l == 10 ? 223 : l == 11 ? 217 : l == 12 ? 211
       : l == 13 ? 199 : l == 14 ? 197 : 193;
}

constexpr bool mod_at_matches() {
  for (int l = 0; l < kMaxMod; ++l)
    if (mod_at(l) != kMods[l]) return false;
  return true;
}
static_assert(mod_at_matches(), "mod_at() and kMods[] list the same moduli");

// x mod m in [0, m) for -2^30 < x < 2^30 (m a compile-time constant after unrolling)
__device__ __forceinline__ int mod_of(int x, int m) {
  const uint32_t bias = (uint32_t)m * ((1u << 30) / (uint32_t)m + 1u);  // multiple of m above 2^30
  return (int)(((uint32_t)x + bias) % (uint32_t)m);
}

// symmetric residue (odd m: [-(m-1)/2, (m-1)/2]; 256: [-128, 127]) of an integer |a| ≤ 2^60 held as
// limbs a = a2·2^40 + a1·2^20 + a0 (a0, a1 in [0, 2^20), a2 signed)
__device__ __forceinline__ int sym_residue(int a2, int a1, int a0, int m) {
  if (m == 256) return (int)(int8_t)(uint8_t)a0;  // low byte, two's complement
  const int c20 = (int)((1u << 20) % (uint32_t)m), c40 = (int)(((uint64_t)1 << 40) % (uint64_t)m);
  const int r = mod_of(a2 * c40 + a1 * c20 + a0, m);  // |·| < 2^29
  return r > (m >> 1) ? r - m : r;
}

// x (|x| ≤ 2^60) rounded to the nearest integer (ties to even) as limbs
__device__ __forceinline__ void limbs(double x, int& a2, int& a1, int& a0) {
  const long long v = __double2ll_rn(x);
  a0 = (int)(v & 0xFFFFF);
  a1 = (int)((v >> 20) & 0xFFFFF);
  a2 = (int)(v >> 40);
}

// e[i] = bias + frexp exponent of max_k |A[i][k]| (0 if the row is zero); an Inf / NaN operand
// latches kErrNonFinite in the device error word (reported by mm_sync_check)
__global__ void row_exp_kernel(const double* __restrict__ A, int64_t lda, int64_t n, int* __restrict__ e,
                               int* __restrict__ err) {
  const double* a = A + (int64_t)blockIdx.x * lda;
  double mx = 0.0;
  int bad = 0;
#pragma unroll 4
  for (int k = threadIdx.x; k < (int)n; k += blockDim.x) {  // n < 2^17 (the emulation's bound)
    const double x = a[k];
    bad |= (__double2hiint(x) & 0x7FF00000) == 0x7FF00000;  // Inf or NaN: all exponent bits set
    mx = fmax(mx, fabs(x));
  }
  if (bad) atomicCAS(err, 0, kErrNonFinite);
  const int64_t i = blockIdx.x;
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
                               int* __restrict__ f, int* __restrict__ err) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= p) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per, r1 = min(n, r0 + rows_per);
  double mx = 0.0;
  int bad = 0;
  for (int64_t k = r0; k < r1; ++k) {
    const double x = B[k * ldb + j];
    bad |= (__double2hiint(x) & 0x7FF00000) == 0x7FF00000;  // Inf or NaN
    mx = fmax(mx, fabs(x));
  }
  if (bad) atomicCAS(err, 0, kErrNonFinite);
  if (mx > 0.0) {
    int ex = 0;
    frexp(mx, &ex);
    atomicMax(f + j, ex + kExpBias);
  }
}

// A residue planes: Ar[(l*mp + i)*kp + k] = a'_ik mod m_l (k >= n or i >= m: 0 — the planes are
// stacked along M in whole 256-row tiles for the batched product); 4 consecutive k per thread
template <int N>
__global__ void residues_a_kernel(const double* __restrict__ A, int64_t lda, int64_t m, int64_t mp, int64_t n,
                                  int64_t kp, const int* __restrict__ e, int beta, int8_t* __restrict__ Ar) {
  const int64_t q4 = kp / 4;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < mp * q4; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = w / q4, k0 = (w % q4) * 4;
    const int sc = i < m ? beta - dec_exp(e[i]) : 0;
    const double s1 = pow2(sc / 2), s2 = pow2(sc - sc / 2);  // scale2, hoisted
    int a2[4], a1[4], a0[4];
#pragma unroll
    for (int c = 0; c < 4; ++c)
      limbs(i < m && k0 + c < n ? A[i * lda + k0 + c] * s1 * s2 : 0.0, a2[c], a1[c], a0[c]);
#pragma unroll
    for (int l = 0; l < N; ++l) {
      uint32_t word = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) word |= (uint32_t)(uint8_t)(int8_t)sym_residue(a2[c], a1[c], a0[c], mod_at(l)) << (8 * c);
      *reinterpret_cast<uint32_t*>(Ar + ((int64_t)l * mp + i) * kp + k0) = word;
    }
  }
}

// B residue planes: Br[(l*kp + k)*pp + j] = b'_kj mod m_l (j >= p or k >= n: 0); 4 consecutive j per thread
template <int N>
__global__ void residues_b_kernel(const double* __restrict__ B, int64_t ldb, int64_t n, int64_t kp, int64_t p,
                                  int64_t pp, const int* __restrict__ f, int beta, int8_t* __restrict__ Br) {
  const int64_t q4 = pp / 4;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < kp * q4; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t k = w / q4, j0 = (w % q4) * 4;
    int a2[4], a1[4], a0[4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int64_t j = j0 + c;
      limbs(j < p && k < n ? scale2(B[k * ldb + j], beta - dec_exp(f[j])) : 0.0, a2[c], a1[c], a0[c]);
    }
#pragma unroll
    for (int l = 0; l < N; ++l) {
      uint32_t word = 0;
#pragma unroll
      for (int c = 0; c < 4; ++c) word |= (uint32_t)(uint8_t)(int8_t)sym_residue(a2[c], a1[c], a0[c], mod_at(l)) << (8 * c);
      *reinterpret_cast<uint32_t*>(Br + ((int64_t)l * kp + k) * pp + j0) = word;
    }
  }
}

// double-double t·M + v (M < 2^24, |v| < 2^24): Horner step of the mixed-radix value
__device__ __forceinline__ void dd_step(double& hi, double& lo, double m, double v) {
  const double p = hi * m;
  const double pe = fma(hi, m, -p);  // hi·m = p + pe exactly
  const double s = p + v;
  const double bb = s - p;
  const double se = (p - (s - bb)) + (v - bb);  // p + v = s + se exactly
  const double l = fma(lo, m, pe + se);
  hi = s + l;
  lo = l - (hi - s);
}

// C[i][j] (+)= 2^-(2β - e_i - f_j) · C'_ij, C' from its residues R_l by Garner + double-double Horner;
// 4 consecutive j per thread (4-byte residue loads, the 4 elements' arithmetic interleaved), pp % 4 == 0
template <int N>
__global__ void __launch_bounds__(256) crt_combine_kernel(const uint8_t* __restrict__ R, int64_t m, int64_t mp,
                                                          int64_t p, int64_t pp, double* __restrict__ C, int64_t ldc,
                                                          const int* __restrict__ e, const int* __restrict__ f,
                                                          int beta_one, const __grid_constant__ CrtTab t) {
  constexpr int G = (N + 2) / 3;                  // digit triples (the last may be short)
  constexpr int kTopBits = 8 * (N - 3 * (G - 1));  // bits of the top triple's value
  constexpr int kPlain = (53 - kTopBits) / 24;    // Horner steps exact in binary64
  const int64_t plane = mp * pp, q4 = (p + 3) / 4;
  for (int64_t w = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; w < m * q4; w += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = w / q4, j0 = (w % q4) * 4;
    const uint32_t* r = reinterpret_cast<const uint32_t*>(R + i * pp + j0);
    uint32_t word[N];
#pragma unroll
    for (int k = 0; k < N; ++k) word[k] = __ldg(r + k * (plane / 4));
    // Garner: v_k = (c_k - Σ_{q<k} v_q P_q) · P_k^-1 mod m_k = c_k·P_k^-1 - Σ_{q<k} v_q·(P_q P_k^-1 mod m_k)
    // mod m_k (tables folded: one reduction per digit), symmetric digits
    int v[4][N];
#pragma unroll
    for (int k = 0; k < N; ++k) {
      const int mk = mod_at(k);
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        int x = (int)((word[k] >> (8 * c)) & 0xFF) * t.pinv[k];
#pragma unroll
        for (int q = 0; q < k; ++q) x -= v[c][q] * t.pmod[q][k];  // |x| < 2^16 + 15·128·256 < 2^20
        const int d = mod_of(x, mk);
        v[c][k] = d > (mk >> 1) ? d - mk : d;  // 256: [-127, 128]; odd: [-(m-1)/2, (m-1)/2]
      }
    }
    const int ei = e[i];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      // triples w_g = v_3g + m_3g (v_3g+1 + m_3g+1 v_3g+2) (|w| < 2^24, exact) in radix M_g = m_3g m_3g+1 m_3g+2:
      // C' = w_0 + M_0 (w_1 + M_1 (w_2 + ...)), Horner exact while below 2^53, double-double below
      int wg[G];
#pragma unroll
      for (int g = 0; g < G; ++g) {
        int acc = 0;
#pragma unroll
        for (int k = 3 * g + 2; k >= 3 * g; --k)
          if (k < N) acc = acc * mod_at(k) + v[c][k];
        wg[g] = acc;
      }
      double hi = (double)wg[G - 1], lo = 0.0;
#pragma unroll
      for (int g = G - 2; g >= 0; --g) {
        const double M = (double)(mod_at(3 * g) * mod_at(3 * g + 1) * mod_at(3 * g + 2));
        if (g >= G - 1 - kPlain) hi = fma(hi, M, (double)wg[g]);
        else dd_step(hi, lo, M, (double)wg[g]);
      }
      const int64_t j = j0 + c;
      if (j < p) {
        const int fj = f[j];
        const double val = (ei && fj) ? scale3(hi + lo, dec_exp(ei) + dec_exp(fj) - 2 * t.beta) : 0.0;
        double* cp = C + i * ldc + j;
        *cp = beta_one ? *cp + val : val;
      }
    }
  }
}

inline int grid_for(int64_t work, int num_sms) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, (int64_t)num_sms * 16));
}

inline size_t up256(size_t x) { return (x + 255) / 256 * 256; }

struct Layout {
  int nmod, beta;
  int64_t mp, kp, pp;  // rows per A / C plane (whole 256-row tiles), K and p padded to 16
  size_t a_bytes, b_bytes, r_bytes, e_bytes, f_bytes, total;
};

bool layout_for(int64_t m, int64_t n, int64_t p, Layout* L) {
  if (!crt_plan(n, &L->nmod, &L->beta)) return false;
  L->mp = (m + 255) / 256 * 256;
  L->kp = (n + 15) / 16 * 16;
  L->pp = (p + 15) / 16 * 16;
  L->a_bytes = up256((size_t)(L->nmod * L->mp * L->kp));
  L->b_bytes = up256((size_t)(L->nmod * L->kp * L->pp));
  L->r_bytes = up256((size_t)(L->nmod * L->mp * L->pp));
  L->e_bytes = up256((size_t)m * 4);
  L->f_bytes = up256((size_t)p * 4);
  L->total = L->a_bytes + L->b_bytes + L->r_bytes + L->e_bytes + L->f_bytes;
  return true;
}

template <int N>
void launch_residues(const double* A, int64_t lda, const double* B, int64_t ldb, int64_t m, int64_t n, int64_t p,
                     const Layout& L, const int* e, const int* f, int8_t* Ar, int8_t* Br, const CrtTab& t, int sms,
                     cudaStream_t s) {
  residues_a_kernel<N><<<grid_for(L.mp * (L.kp / 4), sms), 256, 0, s>>>(A, lda, m, L.mp, n, L.kp, e, t.beta, Ar);
  residues_b_kernel<N><<<grid_for(L.kp * (L.pp / 4), sms), 256, 0, s>>>(B, ldb, n, L.kp, p, L.pp, f, t.beta, Br);
}

template <int N>
void launch_combine(const uint8_t* R, int64_t m, int64_t mp, int64_t p, int64_t pp, double* C, int64_t ldc,
                    const int* e, const int* f, int beta_one, const CrtTab& t, int sms, cudaStream_t s) {
  crt_combine_kernel<N><<<grid_for(m * ((p + 3) / 4), sms), 256, 0, s>>>(R, m, mp, p, pp, C, ldc, e, f, beta_one, t);
}

}  // namespace

int64_t f64_emu_max_n() { return (int64_t)INT32_MAX / (128 * 128); }  // n · 2^14 < 2^31

size_t f64_emu_scratch(int64_t m, int64_t n, int64_t p) {
  Layout L;
  return layout_for(m, n, p, &L) ? L.total : 0;
}

int f64_emu_moduli(int64_t n, int* beta, int* mods) {
  int nm = 0, b = 0;
  if (!crt_plan(n, &nm, &b)) return 0;
  if (beta) *beta = b;
  if (mods)
    for (int l = 0; l < nm; ++l) mods[l] = kMods[l];
  return nm;
}

mm_status gemm_f64_emu(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double* C, int64_t ldc, int beta_one, cudaStream_t s) {
  if (n > f64_emu_max_n())
    return set_err(ctx, MM_ERR_UNSUPPORTED, "MM_F64_EMU: n = %lld exceeds the exact-INT32 bound %lld", (long long)n,
                   (long long)f64_emu_max_n());
  Layout L;
  if (!layout_for(m, n, p, &L))
    return set_err(ctx, MM_ERR_UNSUPPORTED, "MM_F64_EMU: no modulus set for n = %lld", (long long)n);
  mm_status st = ensure_buffer(ctx, &ctx->emu_buf, &ctx->emu_bytes, L.total);
  if (st != MM_OK) return st;
  uint8_t* base = static_cast<uint8_t*>(ctx->emu_buf);
  int8_t* Ar = reinterpret_cast<int8_t*>(base);
  int8_t* Br = reinterpret_cast<int8_t*>(base + L.a_bytes);
  uint8_t* R = base + L.a_bytes + L.b_bytes;
  int* e = reinterpret_cast<int*>(R + L.r_bytes);
  int* f = reinterpret_cast<int*>(R + L.r_bytes + L.e_bytes);
  const CrtTab t = make_tab(L.nmod, L.beta);
  const int sms = ctx->num_sms;
  auto chk = [&](const char* what, int kernels) -> mm_status {
    const cudaError_t ce = cudaGetLastError();
    if (ce != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "MM_F64_EMU %s launch failed: %s", what, cudaGetErrorString(ce));
    ctx->launches += kernels;
    return MM_OK;
  };
  // scales
  row_exp_kernel<<<(unsigned)m, 256, 0, s>>>(A, lda, n, e, ctx->d_err);
  if ((st = chk("row exponents", 1)) != MM_OK) return st;
  if (cudaMemsetAsync(f, 0, (size_t)p * 4, s) != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "MM_F64_EMU memset failed");
  const int64_t rows_per = std::max<int64_t>(64, (n + 63) / 64);
  col_exp_kernel<<<dim3((unsigned)((p + 255) / 256), (unsigned)((n + rows_per - 1) / rows_per)), 256, 0, s>>>(B, ldb, n, p,
                                                                                                           rows_per, f, ctx->d_err);
  if ((st = chk("column exponents", 1)) != MM_OK) return st;
  // residues of the scaled integers
  switch (L.nmod) {
    case 14: launch_residues<14>(A, lda, B, ldb, m, n, p, L, e, f, Ar, Br, t, sms, s); break;
    case 15: launch_residues<15>(A, lda, B, ldb, m, n, p, L, e, f, Ar, Br, t, sms, s); break;
    default: launch_residues<16>(A, lda, B, ldb, m, n, p, L, e, f, Ar, Br, t, sms, s); break;
  }
  if ((st = chk("residues", 2)) != MM_OK) return st;
  // The N exact INT8 products; their epilogue stores C'_l mod m_l as bytes straight into residue
  // plane l (ctx->res_*; an INT32 array + a reduction pass cost 8.7 % of an 8192^3 product).
  // Products of less than two waves of 256-wide tiles run as ONE batched launch — the A planes
  // stacked along M (batch l = rows [l·mp, (l+1)·mp)), each batch reading its own B plane: no N
  // launches of a partial wave each (C2 shape 1.44x, 2048^3 1.24x, 1024^3 1.77x); larger ones as N
  // launches, which the batched form did not beat (4096^3-32768^3: 0.95-0.99x,
  // profiles/ab_emu_batched_r2zz14.txt)
  struct ResetRes {
    mm_ctx* c;
    ~ResetRes() { c->res_mod = 0; c->res_nbat = 0; }
  } reset{ctx};
  const int64_t tiles_one = ((m + 255) / 256) * ((p + 255) / 256);
  bool batched = tiles_one < 2 * (int64_t)(sms / 2);
  if (const char* e = knob("MM_EMU_BATCH")) batched = atoi(e) != 0;  // tuning knob (A/B)
  if (batched) {
    ctx->res_mod = t.m[0];
    ctx->res_nbat = L.nmod;
    for (int l = 0; l < L.nmod; ++l) ctx->res_mods[l] = t.m[l];
    ctx->res_bat_rows = L.mp;
    ctx->res_bat_krows = L.kp;
    st = gemm_ld(ctx, (int64_t)L.nmod * L.mp, L.kp, p, MM_S8_S32, Ar, L.kp, Br, L.pp, R, L.pp, 0, s);
    if (st != MM_OK) return st;
  } else {
    ctx->res_nbat = 1;
    for (int l = 0; l < L.nmod; ++l) {
      ctx->res_mod = t.m[l];
      st = gemm_ld(ctx, m, L.kp, p, MM_S8_S32, Ar + (int64_t)l * L.mp * L.kp, L.kp, Br + (int64_t)l * L.kp * L.pp,
                   L.pp, R + (int64_t)l * L.mp * L.pp, L.pp, 0, s);
      if (st != MM_OK) return st;
    }
  }
  ctx->res_mod = 0;
  ctx->res_nbat = 0;
  // Chinese remaindering, scaling and the binary64 store
  switch (L.nmod) {
    case 14: launch_combine<14>(R, m, L.mp, p, L.pp, C, ldc, e, f, beta_one, t, sms, s); break;
    case 15: launch_combine<15>(R, m, L.mp, p, L.pp, C, ldc, e, f, beta_one, t, sms, s); break;
    default: launch_combine<16>(R, m, L.mp, p, L.pp, C, ldc, e, f, beta_one, t, sms, s); break;
  }
  return chk("CRT combine", 1);
}

}  // namespace mmb
