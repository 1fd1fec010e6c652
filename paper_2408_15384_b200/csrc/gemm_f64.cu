// gemm_f64.cu — C (+)= A·B in IEEE binary64, the paper's own precision
// (`double`), on the FP64 tensor pipe.
//
// sm_100a has no FP64 tcgen05 kind, so the MMA is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) with register accumulators; the
// operand pipeline is still Blackwell-native: TMA 2-D boxes into a
// 128-byte-swizzled shared-memory ring with full/empty mbarriers between one
// producer warp and eight consumer warps ("cache tiling",
// PAPER.md:366-373 prefetching/pipelining, done by TMA instead of the CPU).
//
// CTA tile 128×128, K slab 16 (one 128-B swizzle row of A).  Consumer warp w
// owns a 64×32 sub-tile (2×4 warp grid): 8×4 DMMA tiles, 64 accumulators.
// Fragment loads are conflict-free with the swizzle because each DMMA's four
// k indices are taken from rows {b, b+1, b+4, b+5} of the slab (b ∈ {0,2,8,10}):
// the same four k's for A and B, so each DMMA still adds A[i][k]·B[k][j] over
// its four k's; only which k's are grouped together changes (the sum over all
// k is unchanged up to FP64 rounding order).
// Edges: TMA zero-fills out-of-bounds reads; stores are predicated.
#include "kernels.h"
#include "ptx.cuh"

namespace mmb {

namespace {

constexpr int BM = 128, BN = 128, BK = 16;
constexpr int STAGES = 6;
constexpr int A_BYTES = BM * BK * 8;        // 16 KB, one box {16, 128}
constexpr int BBOX_BYTES = BK * 16 * 8;      // 2 KB, box {16 cols, 16 rows}
constexpr int NBBOX = BN / 16;               // 8 boxes
constexpr int B_BYTES = NBBOX * BBOX_BYTES;  // 16 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int NCONS = 8;                      // consumer warps
constexpr int kThreads = (NCONS + 1) * 32;    // + producer warp
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + 1024;

__global__ void __launch_bounds__(kThreads, 1)
    gemm_f64_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB, GemmArgs args,
                    int tiles_m, int tiles_n, int num_kb) {
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base = (raw_u32 + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_u32);
  const uint32_t sA = base;
  const uint32_t sB = base + STAGES * A_BYTES;
  const uint32_t bar0 = smem_u32(smem + STAGES * STAGE_BYTES);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int num_tiles = tiles_m * tiles_n;
  int* err = args.err;

  if (warp == NCONS && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), NCONS);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == NCONS) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool ok = true;
      for (int t = blockIdx.x; t < num_tiles && ok; t += gridDim.x) {
        const int tm = t % tiles_m, tn = t / tiles_m;  // M fastest: neighbours share B columns
        const int m0 = tm * BM, n0 = tn * BN;
        for (int kb = 0; kb < num_kb; ++kb) {
          if (!mbar_wait(empty_bar(stage), phase ^ 1u, err, 11)) { ok = false; break; }
          mbar_arrive_expect_tx(full_bar(stage), STAGE_BYTES);
          const int k0 = kb * BK;
          tma_load_2d(sA + stage * A_BYTES, &tmA, full_bar(stage), k0, m0);
#pragma unroll
          for (int b = 0; b < NBBOX; ++b)
            tma_load_2d(sB + stage * B_BYTES + b * BBOX_BYTES, &tmB, full_bar(stage), n0 + b * 16, k0);
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
    }
  } else {
    // ---------------------------------------------------------------- DMMA consumers
    const int wm = (int)warp >> 2;  // 0..1 : rows wm*64
    const int wn = (int)warp & 3;   // 0..3 : cols wn*32
    const int g = (int)lane >> 2;   // fragment row / column index 0..7
    const int kk = (int)lane & 3;   // fragment k index 0..3
    const int kofs = (kk & 1) + ((kk >> 1) << 2);  // k within quad: {0,1,4,5}
    // Per-lane smem byte offsets (stage-relative), for quad base 0; quad b adds to k.
    int a_row[8];
#pragma unroll
    for (int mi = 0; mi < 8; ++mi) a_row[mi] = wm * 64 + mi * 8 + g;
    int b_col[4];
#pragma unroll
    for (int ni = 0; ni < 4; ++ni) b_col[ni] = wn * 32 + ni * 8 + g;

    double* C = reinterpret_cast<double*>(args.C);
    const bool vec_ok = ((args.ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(args.C) & 15) == 0);
    int stage = 0;
    uint32_t phase = 0;
    bool ok = true;
    for (int t = blockIdx.x; t < num_tiles && ok; t += gridDim.x) {
      const int tm = t % tiles_m, tn = t / tiles_m;
      double acc[8][4][2];
#pragma unroll
      for (int mi = 0; mi < 8; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

      for (int kb = 0; kb < num_kb; ++kb) {
        if (!mbar_wait(full_bar(stage), phase, err, 12)) { ok = false; break; }
        const uint8_t* pa = smem + stage * A_BYTES;
        const uint8_t* pb = smem + STAGES * A_BYTES + stage * B_BYTES;
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          const int k = ((qd & 1) << 1) + ((qd >> 1) << 3) + kofs;  // quad bases 0,2,8,10
          double af[8], bf[4];
#pragma unroll
          for (int mi = 0; mi < 8; ++mi) {
            const int r = a_row[mi];
            af[mi] = *reinterpret_cast<const double*>(pa + r * 128 + ((((k >> 1) ^ (r & 7))) << 4) + ((k & 1) << 3));
          }
#pragma unroll
          for (int ni = 0; ni < 4; ++ni) {
            const int c = b_col[ni];
            const int cc = c & 15;
            bf[ni] = *reinterpret_cast<const double*>(pb + (c >> 4) * BBOX_BYTES + k * 128 +
                                                      ((((cc >> 1) ^ (k & 7))) << 4) + ((cc & 1) << 3));
          }
#pragma unroll
          for (int mi = 0; mi < 8; ++mi)
#pragma unroll
            for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af[mi], bf[ni]);
        }
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(stage));
        if (++stage == STAGES) { stage = 0; phase ^= 1u; }
      }
      if (!ok) break;
      // epilogue: registers -> global (predicated on the ragged edges)
#pragma unroll
      for (int mi = 0; mi < 8; ++mi) {
        const int64_t row = (int64_t)tm * BM + wm * 64 + mi * 8 + g;
        if (row >= args.M) continue;
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) {
          const int64_t col = (int64_t)tn * BN + wn * 32 + ni * 8 + kk * 2;
          double* dst = C + row * args.ldc + col;
          double v0 = acc[mi][ni][0], v1 = acc[mi][ni][1];
          if (vec_ok && col + 1 < args.N) {
            if (args.beta_one) {
              const double2 o = *reinterpret_cast<const double2*>(dst);
              v0 += o.x;
              v1 += o.y;
            }
            *reinterpret_cast<double2*>(dst) = make_double2(v0, v1);
          } else {
            if (col < args.N) dst[0] = args.beta_one ? dst[0] + v0 : v0;
            if (col + 1 < args.N) dst[1] = args.beta_one ? dst[1] + v1 : v1;
          }
        }
      }
    }
  }
  __syncwarp();
  __syncthreads();
}

}  // namespace

void f64_box_dims(uint32_t* a_box, uint32_t* b_box) {
  a_box[0] = BK;
  a_box[1] = BM;
  b_box[0] = 16;
  b_box[1] = BK;
}

cudaError_t launch_gemm_f64(const CUtensorMap& tmA, const CUtensorMap& tmB, const GemmArgs& a, int num_sms,
                            cudaStream_t s) {
  static bool attr_set = false;
  if (!attr_set) {
    cudaError_t e = cudaFuncSetAttribute(gemm_f64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  const int tiles_m = (int)((a.M + BM - 1) / BM);
  const int tiles_n = (int)((a.N + BN - 1) / BN);
  const int num_tiles = tiles_m * tiles_n;
  const int num_kb = (int)((a.K + BK - 1) / BK);
  int grid = num_tiles < num_sms ? num_tiles : num_sms;
  gemm_f64_kernel<<<grid, kThreads, SMEM_BYTES, s>>>(tmA, tmB, a, tiles_m, tiles_n, num_kb);
  return cudaGetLastError();
}

}  // namespace mmb
