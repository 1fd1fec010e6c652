// synthgen_cuda.cu — the synthgen recipe (synthgen.c) evaluated on the GPU, so large
// inputs (C4: 2 x 512 MiB, C5: 2 x 8 GiB) are created in HBM without a host pass or a
// PCIe copy.  Same counter-based SplitMix64 stream, same mappings,
// bit-for-bit the host generator's output (checked against the host checksums in
// tests/test_synthgen_gpu.py).  Like synthgen.c it holds none of the method's
// arithmetic.  Built with -fmad=false so no multiply-add is contracted.
#include <cuda_runtime.h>
#include <math_constants.h>

#include <cstdint>

namespace {

constexpr uint64_t kGolden = 0x9E3779B97F4A7C15ULL;

__device__ __forceinline__ uint64_t fmix64(uint64_t z) {
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}
__device__ __forceinline__ uint64_t word(uint64_t key, uint64_t idx) { return fmix64(key + (idx + 1) * kGolden); }

// one round-to-nearest-even double -> bf16 (values here are finite, |x| < 16)
__device__ __forceinline__ uint16_t bf16_rne(double x) {
  if (x == 0.0) return signbit(x) ? 0x8000 : 0;
  int e;
  const double m = frexp(x, &e);
  const double r = ldexp(rint(ldexp(m, 8)), e - 8);
  const float f = (float)r;
  return (uint16_t)(__float_as_uint(f) >> 16);
}

__global__ void k_f64(uint64_t key, int64_t N, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)(word(key, (uint64_t)i) >> 11) * 0x1p-52 - 1.0;
}

__global__ void k_i8(uint64_t key, int64_t N, int8_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (int8_t)((int64_t)(((word(key, (uint64_t)i) >> 32) * 255ULL) >> 32) - 127);
}

__global__ void k_exact_f64(uint64_t key, uint64_t K, int64_t N, double* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = (double)((int64_t)(((word(key, (uint64_t)i) >> 32) * K) >> 32) - (int64_t)((K - 1) / 2));
}

__global__ void k_exact_bf16(uint64_t key, uint64_t K, int64_t N, uint16_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = bf16_rne((double)((int64_t)(((word(key, (uint64_t)i) >> 32) * K) >> 32) - (int64_t)((K - 1) / 2)));
}

// Box-Muller on the pair q = i >> 1, as synthgen.c box_muller_at
__global__ void k_bf16_normal(uint64_t key, int64_t N, uint16_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N; i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t q = (uint64_t)i >> 1;
    const uint64_t w1 = fmix64(key + (2 * q + 1) * kGolden);
    const uint64_t w2 = fmix64(key + (2 * q + 2) * kGolden);
    const double u1 = ((double)(w1 >> 12) + 0.5) * 0x1p-52;
    const double u2 = ((double)(w2 >> 12) + 0.5) * 0x1p-52;
    const double r = sqrt(-2.0 * log(u1));
    const double t = 2.0 * CUDART_PI * u2;
    out[i] = bf16_rne((i & 1) ? r * sin(t) : r * cos(t));
  }
}

inline uint64_t host_key(uint64_t seed, uint64_t role) {
  uint64_t z = 4 * seed + role;
  z ^= z >> 30;
  z *= 0xBF58476D1CE4E5B9ULL;
  z ^= z >> 27;
  z *= 0x94D049BB133111EBULL;
  z ^= z >> 31;
  return z;
}

inline int grid_for(int64_t N) {
  int64_t b = (N + 255) / 256;
  return (int)(b > 148 * 32 ? 148 * 32 : (b < 1 ? 1 : b));
}

}  // namespace

extern "C" {

// kind: 0 = f64 U[-1,1), 1 = i8 U{-127..127}, 2 = bf16 N(0,1), 3 = exact f64 (K), 4 = exact bf16 (K)
__attribute__((visibility("default"))) int sgc_generate(int kind, uint64_t seed, uint64_t role, uint64_t K, int64_t rows, int64_t cols, void* out,
                 void* stream) {
  const int64_t N = rows * cols;
  if (N <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const uint64_t key = host_key(seed, role);
  switch (kind) {
    case 0: k_f64<<<grid_for(N), 256, 0, s>>>(key, N, static_cast<double*>(out)); break;
    case 1: k_i8<<<grid_for(N), 256, 0, s>>>(key, N, static_cast<int8_t*>(out)); break;
    case 2: k_bf16_normal<<<grid_for(N), 256, 0, s>>>(key, N, static_cast<uint16_t*>(out)); break;
    case 3: k_exact_f64<<<grid_for(N), 256, 0, s>>>(key, K, N, static_cast<double*>(out)); break;
    case 4: k_exact_bf16<<<grid_for(N), 256, 0, s>>>(key, K, N, static_cast<uint16_t*>(out)); break;
    default: return 2;
  }
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // extern "C"
