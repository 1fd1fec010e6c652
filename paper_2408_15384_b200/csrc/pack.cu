// pack.cu — edge path for operands TMA cannot read in place (base not 16-B
// aligned, or a row pitch that is not a multiple of 16 B): copy
// into a zero-padded, 16-B-pitched buffer.  The padding columns are zeros, so
// they add exactly 0 to every dot product and are never
// stored back.  One thread produces 16 destination bytes (coalesced 16-B
// stores); source reads are byte-granular because the source may be
// arbitrarily aligned.
#include "kernels.h"

namespace mmb {

namespace {

template <int ESZ>
__global__ void pack_pad_kernel(const uint8_t* __restrict__ src, int64_t rows, int64_t cols, int64_t src_ld,
                                uint8_t* __restrict__ dst, int64_t dst_ld) {
  // dst_ld * ESZ is a multiple of 16 by construction.
  const int64_t chunks_per_row = dst_ld * ESZ / 16;
  const int64_t total = rows * chunks_per_row;
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < total; c += (int64_t)gridDim.x * blockDim.x) {
    const int64_t r = c / chunks_per_row;
    const int64_t byte0 = (c - r * chunks_per_row) * 16;
    const uint8_t* s = src + r * src_ld * ESZ;
    const int64_t row_bytes = cols * ESZ;
    alignas(16) uint8_t buf[16];
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int64_t b = byte0 + i;
      buf[i] = b < row_bytes ? s[b] : (uint8_t)0;
    }
    *reinterpret_cast<uint4*>(dst + r * dst_ld * ESZ + byte0) = *reinterpret_cast<const uint4*>(buf);
  }
}

}  // namespace

cudaError_t launch_pack_pad(const void* src, int64_t rows, int64_t cols, int64_t src_ld, void* dst, int64_t dst_ld,
                            int esize, cudaStream_t s) {
  const int64_t total = rows * (dst_ld * esize / 16);
  if (total <= 0) return cudaSuccess;
  int64_t blocks = (total + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  const auto* sp = static_cast<const uint8_t*>(src);
  auto* dp = static_cast<uint8_t*>(dst);
  switch (esize) {
    case 1: pack_pad_kernel<1><<<(int)blocks, 256, 0, s>>>(sp, rows, cols, src_ld, dp, dst_ld); break;
    case 2: pack_pad_kernel<2><<<(int)blocks, 256, 0, s>>>(sp, rows, cols, src_ld, dp, dst_ld); break;
    case 4: pack_pad_kernel<4><<<(int)blocks, 256, 0, s>>>(sp, rows, cols, src_ld, dp, dst_ld); break;
    case 8: pack_pad_kernel<8><<<(int)blocks, 256, 0, s>>>(sp, rows, cols, src_ld, dp, dst_ld); break;
    default: return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

}  // namespace mmb
