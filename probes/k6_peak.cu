// k6_peak.cu — MMA-only peak probes (kernel K6): measured operations per
// clock per SM of the instructions the product kernels issue, so the "clock-normalised" roofline
// denominator is a measurement, not the spec sheet.  Measurement infrastructure for bench.py; not
// part of the product path.
//
//   BF16: tcgen05.mma.cta_group::2.kind::f16, M=256 N=256 K=16, FP32 accumulators in TMEM
//   INT8: tcgen05.mma.cta_group::2.kind::i8,  M=256 N=256 K=32, INT32 accumulators in TMEM
//   FP64: mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4), register accumulators, 16 warps per SM
//
// Every SM runs the instruction back to back on operands already in shared memory / registers (no
// loads, no epilogue); each CTA times its own loop with clock64 and globaltimer.  Result per SM:
// flop / cycles; the effective SM clock = cycles / ns.  Operands are zero (shared memory is zeroed):
// the count of operations per clock does not depend on the values, the power draw (and so the clock
// reached) does — the clock is reported separately and is not used as a peak.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "ptx.cuh"

using namespace mmb;

namespace {

constexpr int kPairN = 256, kPairM = 256;

template <bool I8>
__global__ void __launch_bounds__(128, 1) k6_tc_kernel(int iters, unsigned long long* out /* per CTA: cycles, ns */) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  const uint32_t raw = smem_u32(smem_raw);
  const uint32_t base = (raw + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw);
  const uint32_t sA = base;                // 128 rows x 128 B (K-major, SW128)
  const uint32_t sB = base + 16384;        // 2 boxes of 128 B x BK rows (MN-major, SW128)
  const uint32_t bar = smem_u32(smem + 32768);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(smem + 32768 + 64);
  for (int i = threadIdx.x; i < 32768 / 16; i += blockDim.x) reinterpret_cast<uint4*>(smem)[i] = make_uint4(0, 0, 0, 0);
  const uint32_t warp = warp_id(), lane = lane_id();
  const uint32_t rank = __shfl_sync(0xffffffffu, cluster_ctarank(), 0);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    fence_mbar_init();
  }
  fence_proxy_async_smem();
  if (warp == 1) tmem_alloc<2>(smem_u32(tmem_slot), 512);
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  const uint32_t tmem = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  if (warp == 1 && rank == 0) {
    constexpr uint32_t IDESC = ((I8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                               ((uint32_t)(kPairN >> 3) << 17) | ((uint32_t)(kPairM >> 4) << 24);
    constexpr int BOX_BYTES = 64 * 128 * (I8 ? 2 : 1);  // BK rows x 128 B (BK = 128 B of K)
    const uint64_t adesc = umma_desc_sw128(sA, 16, 1024);
    const uint64_t bdesc = umma_desc_sw128(sB, BOX_BYTES, 1024);
    __syncwarp();
    const uint64_t c0 = clock64();
    const uint64_t t0 = globaltimer_ns();
    for (int i = 0; i < iters; ++i)
      if (lane == 0) tc_mma<2, I8>(tmem + (uint32_t)(i & 1) * 256u, adesc, bdesc, IDESC, i > 1 ? 1u : 0u);
    if (lane == 0) tc_commit<2>(bar, 0x3);
    __syncwarp();
    mbar_wait(bar, 0, nullptr, 0);
    const uint64_t c1 = clock64();
    const uint64_t t1 = globaltimer_ns();
    if (lane == 0) {
      out[2 * blockIdx.x] = c1 - c0;
      out[2 * blockIdx.x + 1] = t1 - t0;
    }
  } else if (warp == 1 && rank == 1) {
    mbar_wait(bar, 0, nullptr, 0);  // the leader's commit arrives here too (multicast)
  }
  tc_fence_before();
  cluster_sync();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<2>(tmem, 512);
}

// 16 warps per SM, each DMMA.8x8x4 back to back on 8 independent accumulator pairs.
__global__ void __launch_bounds__(512, 1) k6_dmma_kernel(int iters, unsigned long long* out, double* sink) {
  double acc[8][2];
#pragma unroll
  for (int i = 0; i < 8; ++i) acc[i][0] = acc[i][1] = 0.0;
  const double a = 1.0 + 1e-3 * threadIdx.x, b = 1.0 - 1e-3 * threadIdx.x;
  __syncthreads();
  const uint64_t c0 = clock64();
  const uint64_t t0 = globaltimer_ns();
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) dmma_8x8x4(acc[i][0], acc[i][1], a, b);
  }
  __syncthreads();
  const uint64_t c1 = clock64();
  const uint64_t t1 = globaltimer_ns();
  double s = 0;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += acc[i][0] + acc[i][1];
  if (s == 12345.678) sink[0] = s;  // keep the accumulators live
  if (threadIdx.x == 0) {
    out[2 * blockIdx.x] = c1 - c0;
    out[2 * blockIdx.x + 1] = t1 - t0;
  }
}

}  // namespace

extern "C" {

// kind: 0 = BF16 (kind::f16), 1 = INT8 (kind::i8), 2 = FP64 (DMMA).  Runs `reps` launches over all
// SMs and reports the best launch: *flop_per_clk_sm (per SM, median over CTAs), *clock_mhz (median
// effective SM clock over CTAs), *tflops (whole GPU: SMs x flop/clk x clock).  Returns 0 on success.
__attribute__((visibility("default"))) int k6_run(int kind, int iters, int reps, double* flop_per_clk_sm,
                                                  double* clock_mhz, double* tflops) {
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int ctas = kind == 2 ? sms : (sms / 2) * 2;
  unsigned long long* d_out = nullptr;
  double* d_sink = nullptr;
  if (cudaMalloc(&d_out, sizeof(unsigned long long) * 2 * ctas) != cudaSuccess) return 1;
  cudaMalloc(&d_sink, sizeof(double));
  const int smem = 32768 + 1024 + 1024;
  double best = 0, best_clk = 0;
  std::vector<unsigned long long> h(2 * ctas);
  for (int r = 0; r < reps; ++r) {
    cudaError_t e;
    if (kind == 2) {
      k6_dmma_kernel<<<ctas, 512>>>(iters, d_out, d_sink);
      e = cudaGetLastError();
    } else {
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(ctas, 1, 1);
      cfg.blockDim = dim3(128, 1, 1);
      cfg.dynamicSmemBytes = smem;
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = 2;
      attr[0].val.clusterDim.y = 1;
      attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr;
      cfg.numAttrs = 1;
      if (kind == 0) {
        cudaFuncSetAttribute(k6_tc_kernel<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&cfg, k6_tc_kernel<false>, iters, d_out);
      } else {
        cudaFuncSetAttribute(k6_tc_kernel<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
        e = cudaLaunchKernelEx(&cfg, k6_tc_kernel<true>, iters, d_out);
      }
    }
    if (e != cudaSuccess || cudaDeviceSynchronize() != cudaSuccess) {
      cudaFree(d_out);
      cudaFree(d_sink);
      return 2;
    }
    cudaMemcpy(h.data(), d_out, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    std::vector<double> per_sm, clk;
    for (int c = 0; c < ctas; ++c) {
      const double cyc = (double)h[2 * c], ns = (double)h[2 * c + 1];
      if (kind != 2 && (c & 1)) continue;  // the pair's leader timed the pair's MMAs
      if (cyc <= 0 || ns <= 0) continue;
      double flop;
      if (kind == 2) flop = 2.0 * 8 * 8 * 4 * 8.0 * iters * 16;         // 16 warps x 8 DMMAs per iteration
      else flop = 2.0 * kPairM * kPairN * (kind == 0 ? 16 : 32) * iters / 2;  // per SM of the pair
      per_sm.push_back(flop / cyc);
      clk.push_back(cyc / ns * 1e3);
    }
    if (per_sm.empty()) continue;
    std::sort(per_sm.begin(), per_sm.end());
    std::sort(clk.begin(), clk.end());
    const double med = per_sm[per_sm.size() / 2];
    if (med > best) {
      best = med;
      best_clk = clk[clk.size() / 2];
    }
  }
  cudaFree(d_out);
  cudaFree(d_sink);
  *flop_per_clk_sm = best;
  *clock_mhz = best_clk;
  *tflops = best * sms * best_clk * 1e6 / 1e12;
  return best > 0 ? 0 : 3;
}

}  // extern "C"
