// gemm_tc.cu — C = A·B on the 5th-generation tensor cores (tcgen05) for
//   BF16 × BF16 → FP32  (kind::f16, FP32 accumulators in TMEM)
//   INT8 × INT8 → INT32 (kind::i8,  INT32 accumulators in TMEM)
//
// The operation is PAPER.md:56-60 (§III); A m×n and B n×p are row-major
// (PAPER.md:87).  What the paper does on a CPU with cache tiling
// and row-parallel threads is done here as:
//   * tiles of C (128·CG × 256·NT) walked by a persistent grid of CTA clusters
//     in grouped-raster waves (sched.cuh); above 96 MB of operands a wave
//     barrier keeps the k-phase of a wave aligned so its tiles share A/B slabs
//     in L2;
//   * K-slabs of A (K-major) and B (row-major = N-major, consumed as an
//     MN-major UMMA operand, so B's "columns" need no transpose)
//     staged by TMA into 128-byte-swizzled shared memory (KA swizzle atoms of
//     K per stage), full/empty mbarriers between the producer warp and the MMA
//     warp;
//   * one thread issues tcgen05.mma into TMEM: NT = 1, two 256-column
//     accumulators (the epilogue of tile j overlaps the mainloop of tile j+1);
//     NT = 2, one 512-column accumulator of two regions released one by one;
//   * CG = 2: a CTA pair (cluster of 2) runs one M=256 MMA; each CTA stages
//     its own 128 rows of A and half of B's columns; the leader issues and
//     commits to both.  MC = 2 (knob): two pairs share B slabs by multicast;
//   * epilogue: tcgen05.ld -> registers -> 128B-swizzled staging -> TMA store;
//     a split last wave (sched.cuh modes) either adds partial slabs in a fixed
//     order or, by default, adds exact K halves into C with TMA reduce-add;
//   * edges (ragged m, n, p): TMA zero-fills out-of-bounds boxes (zeros add
//     exactly 0 to every sum) and clips out-of-bounds stores;
//   * INT8 only, for MM_F64_EMU (f64_emu.cu): the epilogue can store C mod m as bytes, and one
//     launch can run a batch of products stacked along M, each with its own B rows and modulus
//     (GemmArgs::res_m / bat_rows).
//
// Warp roles (320 threads): warp 0 = TMA producer, warp 1 = TMEM allocator +
// MMA issuer, warps 2..9 = epilogue (two per TMEM lane quarter).
// Programmatic dependent launch: only the prologue overlaps the previous kernel
// in the stream; griddepcontrol.wait precedes every global access (the producer
// before its first load, the epilogue warps before zeroing a reduce-add tail).
#include <algorithm>
#include <atomic>
#include <cstdlib>

#include "kernels.h"
#include "knobs.h"
#include "ptx.cuh"
#include "sched.cuh"

namespace mmb {

namespace {

constexpr int kThreads = 320;  // warp 0 TMA producer, warp 1 TMEM + MMA issuer, warps 2..9 epilogue
constexpr int kBN = 256;  // MMA N (columns of C per tile)

// KA: 128-B swizzle atoms of K per stage (2: twice the MMAs per barrier wait and commit)
template <bool I8, int CG, int NT, int MC = 1, int KA = 1>
struct TcCfg {
  static constexpr int ESZ = I8 ? 1 : 2;
  static constexpr int BKA = 128 / ESZ;       // K elements per 128-B swizzle atom (one A box)
  static constexpr int BK = BKA * KA;         // K elements per stage
  static constexpr int UK = I8 ? 32 : 16;     // K per tcgen05.mma
  static constexpr int KSTEPS = BK / UK;      // 4 per atom
  static constexpr int KPA = BKA / UK;        // K steps per atom
  static constexpr int BM = 128;              // rows of A per CTA
  static constexpr int TILE_N = kBN * NT;     // columns of C per tile (NT accumulators of N=256)
  static constexpr int NBUF = (NT == 1) ? 2 : 1;  // TMEM accumulator buffers: NBUF * TILE_N = 512 columns
  static constexpr int BN_CTA = kBN / CG;     // columns of B per CTA per MMA region
  static constexpr int BOXN = 128 / ESZ;      // columns per TMA box of B (128 B)
  static constexpr int NBOX = BN_CTA / BOXN;  // boxes per region
  static constexpr int A_ATOM = BM * 128;     // one A box
  static constexpr int A_BYTES = A_ATOM * KA;
  static constexpr int BOX_BYTES = BK * 128;
  static constexpr int REGION_BYTES = NBOX * BOX_BYTES;
  static constexpr int B_BYTES = NT * REGION_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = KA == 2 ? 3 : ((CG == 1 || NT == 2) ? 4 : 6);
  static constexpr int EPI_BYTES = 8 * 32 * 128;  // epilogue staging: 8 warps x (32 rows x 128 B)
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + EPI_BYTES + 1024 /*barriers*/ + 1024 /*align slack*/;
  static constexpr int M_MMA = 128 * CG;
  // MC = 2: a cluster of two CTA pairs stacked along M (tile M_MMA*MC rows) shares every B slab:
  // each pair loads half of the slab's K rows and multicasts them into both pairs' shared memory.
  static constexpr int M_TILE = M_MMA * MC;
  static constexpr int BKB = BK / MC;               // K rows per TMA box of B
  static constexpr int B_PART = BOX_BYTES / MC;     // bytes of one such box
  // Instruction descriptor: c_format [4,6), a_format [7,10), b_format [10,13),
  // a_major [15] = K, b_major [16] = MN, N>>3 at [17,23), M>>4 at [24,29).
  static constexpr uint32_t IDESC = ((I8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                                    ((uint32_t)(kBN >> 3) << 17) | ((uint32_t)(M_MMA >> 4) << 24);
  // N-half tail items (sched.nhalf): the pair's MMA is N = 128, each CTA stages 64 columns of B
  // (bf16: one 128-B box of the regular map; int8: a 64-B box through a SWIZZLE_64B map)
  static constexpr uint32_t IDESC_H = ((I8 ? 2u : 1u) << 4) | (1u << 7) | (1u << 10) | (0u << 15) | (1u << 16) |
                                      ((uint32_t)((kBN / 2) >> 3) << 17) | ((uint32_t)(M_MMA >> 4) << 24);
  static constexpr int HB_BYTES = BK * 64 * ESZ;  // one CTA's 64 columns of B per stage
};

__device__ __forceinline__ void store_row32(uint32_t* __restrict__ C, int64_t ldc, int64_t row, int64_t col0,
                                            int64_t M, int64_t N, const uint32_t (&v)[32], bool vec_ok) {
  if (row >= M) return;
  uint32_t* dst = C + row * ldc + col0;
  if (vec_ok && col0 + 32 <= N) {
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
      asm volatile("st.global.v4.b32 [%0], {%1, %2, %3, %4};" ::"l"(dst + i), "r"(v[i]), "r"(v[i + 1]), "r"(v[i + 2]),
                   "r"(v[i + 3])
                   : "memory");
    }
  } else {
#pragma unroll
    for (int i = 0; i < 32; ++i)
      if (col0 + i < N) dst[i] = v[i];
  }
}

// Partial slabs are stored warp-chunk-contiguous: uint4 element (chunk c, warp q, vector i,
// lane l) at ((c*4 + q)*8 + i)*32 + l, so a warp's 32 rows x 32 columns of one chunk are
// 4 KB in one piece (one bulk copy) and each vector i is one coalesced 512-B request.
__device__ __forceinline__ size_t slab_index(int c, int q, int i, int l) { return ((size_t)(c * 4 + q) * 8 + i) * 32 + l; }

template <bool I8>
__device__ __forceinline__ void add_words(uint32_t (&v)[32], const uint4 (&w)[8]) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const uint32_t x[4] = {w[i].x, w[i].y, w[i].z, w[i].w};
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      if constexpr (I8) v[4 * i + u] = (uint32_t)((int32_t)v[4 * i + u] + (int32_t)x[u]);
      else v[4 * i + u] = __float_as_uint(__uint_as_float(v[4 * i + u]) + __uint_as_float(x[u]));
    }
  }
}

template <bool I8>
__device__ __forceinline__ void add_regs(uint32_t (&v)[32], const uint32_t (&o)[32]) {
#pragma unroll
  for (int i = 0; i < 32; ++i) {
    if constexpr (I8) v[i] = (uint32_t)((int32_t)v[i] + (int32_t)o[i]);
    else v[i] = __float_as_uint(__uint_as_float(v[i]) + __uint_as_float(o[i]));
  }
}

template <bool I8>
__device__ __forceinline__ void add32(uint32_t (&v)[32], const uint4* __restrict__ src /* = slab + slab_index(c,q,0,l) */) {
  uint4 w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) w[i] = ld_cg_u4(src + i * 32);  // 8 independent loads in flight
  add_words<I8>(v, w);
}

template <bool I8, int CG, int NT, int MC, int KA>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                   const __grid_constant__ CUtensorMap tmC, const __grid_constant__ CUtensorMap tmBh, GemmArgs args,
                   WorkSched sched) {
  using Cfg = TcCfg<I8, CG, NT, MC, KA>;
  const uint64_t tr_entry = args.trace ? globaltimer_ns() : 0;
  // clock meter (mm_clock_meter): SM cycles and nanoseconds over this CTA's life
  // (held in registers: storing them at entry raised the BF16 pair kernel from 151 to 160 registers)
  uint64_t clk_c0 = 0, clk_t0 = 0;
  if (args.clk && threadIdx.x == 0) {
    clk_c0 = clock64();
    clk_t0 = globaltimer_ns();
  }
  // timeline (MM_TRACE): per CTA, items 0..7: MMA first issue / last issue, epilogue start / end
  unsigned long long* tl = args.trace ? args.trace + 4096 * 16 + (size_t)blockIdx.x * 32 : nullptr;
  extern __shared__ uint8_t smem_raw[];
  // 1024-B alignment (SWIZZLE_128B atoms) of the operand ring.
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base = (raw_u32 + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_u32);
  const uint32_t sA = base;
  const uint32_t sB = base + Cfg::STAGES * Cfg::A_BYTES;
  const uint32_t sEpi = base + Cfg::STAGES * Cfg::STAGE_BYTES;  // 1024-aligned (SWIZZLE_128B staging)
  uint8_t* bar_area = smem + Cfg::STAGES * Cfg::STAGE_BYTES + Cfg::EPI_BYTES;
  const uint32_t bar0 = smem_u32(bar_area);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (Cfg::STAGES + s); };
  auto tfull_bar = [&](int a) { return bar0 + 8u * (2 * Cfg::STAGES + a); };
  auto tempty_bar = [&](int a) { return bar0 + 8u * (2 * Cfg::STAGES + 2 + a); };
  auto land_bar = [&](int q) { return bar0 + 8u * (2 * Cfg::STAGES + 4 + q); };
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(bar_area + 8 * (2 * Cfg::STAGES + 12));
  volatile unsigned* tick_slot = reinterpret_cast<volatile unsigned*>(bar_area + 8 * (2 * Cfg::STAGES + 13));
  static_assert(8 * (2 * Cfg::STAGES + 14) <= 1024, "barrier area");

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  // warp-uniform by construction (__shfl_sync): lets the compiler keep role branches and operand
  // arithmetic in uniform registers (no per-instruction waterfalls around tcgen05 / TMA operands)
  const uint32_t crank = (CG == 2) ? __shfl_sync(0xffffffffu, cluster_ctarank(), 0) : 0u;  // rank in the cluster
  const uint32_t rank = crank & (uint32_t)(CG - 1);            // rank in the CTA pair
  const uint32_t pair = crank / (uint32_t)CG;                   // pair index along M (MC = 2)
  const uint32_t leader = crank - rank;                         // the pair's MMA-issuing CTA
  const int cl = (CG == 2) ? (int)cluster_id_x() : (int)blockIdx.x;
  const int num_kb = sched.num_kb;
  int* err = args.err;

  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
    if (args.c_tma) tma_prefetch_desc(&tmC);
    for (int s = 0; s < Cfg::STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      mbar_init(empty_bar(s), MC);  // one commit from the leader of every pair reading this slot
    }
    for (int a = 0; a < 2; ++a) {  // NT=1: two accumulators; NT=2: one, released region by region
      mbar_init(tfull_bar(a), 1);   // (each release: all 8 epilogue warps of both CTAs)
      mbar_init(tempty_bar(a), 8 * CG);
    }
    for (int qq = 0; qq < 8; ++qq) mbar_init(land_bar(qq), 1);
    fence_mbar_init();
  }
  if (warp == 1) tmem_alloc<CG>(smem_u32(tmem_slot), 512);
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = __shfl_sync(0xffffffffu, *tmem_slot, 0);
  // optional timeline (MM_TRACE=1): per CTA ns spent waiting, by role
  uint64_t tr_barrier = 0, tr_empty = 0, tr_tempty = 0, tr_full = 0, tr_tfull = 0, tr_drain = 0;
  uint64_t tr_c[5] = {0, 0, 0, 0, 0};  // epilogue per-chunk cycles: ld-wait, st.shared, fence, store, chunks
  const uint64_t tr_t0 = args.trace ? globaltimer_ns() : 0;
  const uint64_t tr_clk0 = args.trace ? clock64() : 0;

  if (warp == 0) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool ok = true;
      int t, kb0, kb1;
      // L2 priorities (large operands): the A panels of a raster group are re-read by every
      // wave of the group, the B slabs only within one wave -> keep A, stream B.
      // l2_hint bit 0: A evict_last; bit 1: B evict_first (else evict_normal)
      const uint64_t pol_a = (args.l2_hint & 1) ? l2_policy_evict_last() : l2_policy_evict_normal();
      const uint64_t pol_b = (args.l2_hint & 2) ? l2_policy_evict_first() : l2_policy_evict_normal();
      // Programmatic dependent launch: everything above (barrier init, TMEM allocation, tensor-map
      // prefetch) overlapped the previous kernel in the stream; no global memory is touched before
      // it has completed (the MMA and epilogue only run on data loaded after this wait).
      pdl_wait();
      if (args.trace) args.trace[(size_t)blockIdx.x * 16 + 15] = globaltimer_ns();
      for (int j = 0; ok && sched.item(cl, j, t, kb0, kb1); ++j) {
        // Wave barrier: start item j only when every CTA has issued all loads of its
        // item j-1, so the tiles of a wave walk K in step and share A/B slabs in L2.
        // Soft (bounded, abandoned on time-out): no CTA ever depends on another being resident.
        const uint64_t tb0 = args.trace ? globaltimer_ns() : 0;
        if (args.wave_sync && j > 0 && j <= sched.W) soft_wave_wait(args.sync, (unsigned)j * gridDim.x);
        if (args.trace) tr_barrier += globaltimer_ns() - tb0;
        int tm, tn;
        sched.tile_coords(t, tm, tn);
        const int hf = sched.half_of(cl, j);  // N half of a tail tile, or -1
        // (diagnostics, MM_DEBUG bit 1: every tile reads the first tile's operands -> L2 hits only)
        const int m0 = ((args.debug & 2) ? 0 : tm * Cfg::M_TILE) + (int)pair * Cfg::M_MMA + (int)rank * Cfg::BM;
        const int n0 = ((args.debug & 2) ? 0 : tn * Cfg::TILE_N) + (int)rank * Cfg::BN_CTA;  // + rr * kBN for region rr
        // batched residue products (MM_F64_EMU): this tile's batch reads its own B rows
        const int kbat = args.bat_rows ? (tm * Cfg::M_TILE / args.bat_rows) * args.bat_krows : 0;
        for (int kb = kb0; kb < kb1; ++kb) {
          const uint64_t te0 = args.trace ? globaltimer_ns() : 0;
          if (!mbar_wait(empty_bar(stage), phase ^ 1u, err, 1)) { ok = false; break; }
          if (args.trace) tr_empty += globaltimer_ns() - te0;
          const uint32_t sa = sA + stage * Cfg::A_BYTES;
          const uint32_t sb = sB + stage * Cfg::B_BYTES;
          const int k0 = kb * Cfg::BK;
          if (args.debug & 1) {
            // diagnostics: no operand traffic at all (MMA on whatever is in the slot)
            if (rank == 0) mbar_arrive(full_bar(stage));
          } else if constexpr (CG == 1) {
            mbar_arrive_expect_tx(full_bar(stage), Cfg::STAGE_BYTES);
            if (args.l2_hint) {
#pragma unroll
              for (int a = 0; a < KA; ++a)
                tma_load_2d_hint(sa + a * Cfg::A_ATOM, &tmA, full_bar(stage), k0 + a * Cfg::BKA, m0, pol_a);
#pragma unroll
              for (int rb = 0; rb < NT * Cfg::NBOX; ++rb)
                tma_load_2d_hint(sb + rb * Cfg::BOX_BYTES, &tmB, full_bar(stage),
                                 n0 + (rb / Cfg::NBOX) * kBN + (rb % Cfg::NBOX) * Cfg::BOXN, k0 + kbat, pol_b);
            } else {
#pragma unroll
              for (int a = 0; a < KA; ++a) tma_load_2d(sa + a * Cfg::A_ATOM, &tmA, full_bar(stage), k0 + a * Cfg::BKA, m0);
#pragma unroll
              for (int rb = 0; rb < NT * Cfg::NBOX; ++rb)
                tma_load_2d(sb + rb * Cfg::BOX_BYTES, &tmB, full_bar(stage),
                            n0 + (rb / Cfg::NBOX) * kBN + (rb % Cfg::NBOX) * Cfg::BOXN, k0 + kbat);
            }
          } else if constexpr (MC == 2) {
            // A: this CTA's own 128 rows.  B: this pair's half of the K rows of each box, multicast
            // to the same-rank CTA of both pairs (which need the same B columns).
            const uint32_t leader_full = mapa_shared(full_bar(stage), leader);
            if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), 2 * Cfg::STAGE_BYTES);
#pragma unroll
            for (int a = 0; a < KA; ++a)
              tma_load_2d_pair(sa + a * Cfg::A_ATOM, &tmA, leader_full, k0 + a * Cfg::BKA, m0);
            const uint16_t mask = (uint16_t)((1u << rank) | (1u << (rank + 2)));
#pragma unroll
            for (int rb = 0; rb < NT * Cfg::NBOX; ++rb)
              tma_load_2d_pair_mc(sb + rb * Cfg::BOX_BYTES + pair * Cfg::B_PART, &tmB, leader_full,
                                  n0 + (rb / Cfg::NBOX) * kBN + (rb % Cfg::NBOX) * Cfg::BOXN,
                                  k0 + kbat + (int)pair * Cfg::BKB, mask);
          } else if (NT == 1 && hf >= 0) {
            // N-half tail item: this CTA's 128 rows of A, and its 64 of the half's 128 columns of B
            const uint32_t leader_full = mapa_shared(full_bar(stage), 0);
            if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), 2 * (Cfg::A_BYTES + Cfg::HB_BYTES));
#pragma unroll
            for (int a = 0; a < KA; ++a)
              tma_load_2d_pair(sa + a * Cfg::A_ATOM, &tmA, leader_full, k0 + a * Cfg::BKA, m0);
            tma_load_2d_pair(sb, &tmBh, leader_full, tn * Cfg::TILE_N + hf * (kBN / 2) + (int)rank * (kBN / 4), k0 + kbat);
          } else {
            const uint32_t leader_full = mapa_shared(full_bar(stage), 0);
            if (rank == 0) mbar_arrive_expect_tx(full_bar(stage), 2 * Cfg::STAGE_BYTES);
            if (args.l2_hint) {
#pragma unroll
              for (int a = 0; a < KA; ++a)
                tma_load_2d_pair_hint(sa + a * Cfg::A_ATOM, &tmA, leader_full, k0 + a * Cfg::BKA, m0, pol_a);
#pragma unroll
              for (int rb = 0; rb < NT * Cfg::NBOX; ++rb)
                tma_load_2d_pair_hint(sb + rb * Cfg::BOX_BYTES, &tmB, leader_full,
                                      n0 + (rb / Cfg::NBOX) * kBN + (rb % Cfg::NBOX) * Cfg::BOXN, k0 + kbat, pol_b);
            } else {
#pragma unroll
              for (int a = 0; a < KA; ++a)
                tma_load_2d_pair(sa + a * Cfg::A_ATOM, &tmA, leader_full, k0 + a * Cfg::BKA, m0);
#pragma unroll
              for (int rb = 0; rb < NT * Cfg::NBOX; ++rb)
                tma_load_2d_pair(sb + rb * Cfg::BOX_BYTES, &tmB, leader_full,
                                 n0 + (rb / Cfg::NBOX) * kBN + (rb % Cfg::NBOX) * Cfg::BOXN, k0 + kbat);
            }
          }
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
        }
        if (args.wave_sync && j < sched.W) red_release_gpu_add(args.sync, 1u);
      }
      pdl_launch_dependents();  // all loads issued: the next launch may start its prologue
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------------- MMA issuer (leader CTA)
    // The whole warp runs the loop (barrier waits, descriptor arithmetic: warp-uniform, so the
    // compiler keeps them in uniform registers); lane 0 alone issues the MMAs and commits.
    // Issuing from a divergent single-lane branch made every tcgen05.mma a waterfall of
    // ELECT / R2UR.BROADCAST / BRA.U.ANY around its operands.
    if (rank == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool ok = true;
      int t, kb0, kb1;
      // MMAs of k-block kb of this tile into accumulator region(s) [r0, r1)
      auto issue = [&](uint32_t d_tmem, int stg, bool first_kb, int r0, int r1) {
        const uint32_t sa = sA + stg * Cfg::A_BYTES;
        const uint32_t sb = sB + stg * Cfg::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < Cfg::KSTEPS; ++kk) {
          // A: K-major SW128, rows 128 B apart, 8-row groups 1024 B apart (SBO); K step = 32 B.
          const uint64_t adesc = umma_desc_sw128(sa + (kk / Cfg::KPA) * Cfg::A_ATOM + (kk % Cfg::KPA) * 32, 16, 1024);
#pragma unroll
          for (int rr = 0; rr < NT; ++rr) {
            if (rr < r0 || rr >= r1) continue;
            // B: MN-major SW128, 128-B (BOXN-column) blocks BOX_BYTES apart (LBO), 8-row k groups 1024 B (SBO).
            const uint64_t bdesc =
                umma_desc_sw128(sb + rr * Cfg::REGION_BYTES + kk * Cfg::UK * 128, Cfg::BOX_BYTES, 1024);
            tc_mma_warp<CG, I8>(d_tmem + rr * kBN, adesc, bdesc, Cfg::IDESC, (!first_kb || kk != 0) ? 1u : 0u);
          }
        }
      };
      // MMAs of one k-block of an N-half tail item (pair N = 128) into accumulator `d_tmem`
      auto issue_half = [&](uint32_t d_tmem, int stg, bool first_kb) {
        const uint32_t sa = sA + stg * Cfg::A_BYTES;
        const uint32_t sb = sB + stg * Cfg::B_BYTES;
#pragma unroll
        for (int kk = 0; kk < Cfg::KSTEPS; ++kk) {
          const uint64_t adesc = umma_desc_sw128(sa + (kk / Cfg::KPA) * Cfg::A_ATOM + (kk % Cfg::KPA) * 32, 16, 1024);
          // B: MN-major, one 64-column block per CTA: bf16 rows of 128 B (SW128), int8 rows of 64 B (SW64)
          const uint64_t bdesc = I8 ? umma_desc_sw64(sb + kk * Cfg::UK * 64, Cfg::HB_BYTES, 512)
                                    : umma_desc_sw128(sb + kk * Cfg::UK * 128, Cfg::BOX_BYTES, 1024);
          tc_mma_warp<CG, I8>(d_tmem, adesc, bdesc, Cfg::IDESC_H, (!first_kb || kk != 0) ? 1u : 0u);
        }
      };
      auto wait_tempty = [&](int a, uint32_t parity) {
        const uint64_t tt0 = args.trace ? globaltimer_ns() : 0;
        const bool r = CG == 2 ? mbar_wait_cluster(tempty_bar(a), parity, err, 2) : mbar_wait(tempty_bar(a), parity, err, 2);
        if (args.trace) tr_tempty += globaltimer_ns() - tt0;
        tc_fence_after();
        return __all_sync(0xffffffffu, r) != 0;
      };
      auto wait_full = [&](int stg, uint32_t ph) {
        const uint64_t tf0 = args.trace ? globaltimer_ns() : 0;
        const bool r = mbar_wait(full_bar(stg), ph, err, 3);
        if (args.trace) tr_full += globaltimer_ns() - tf0;
        tc_fence_after();
        return __all_sync(0xffffffffu, r) != 0;
      };
      for (int j = 0; ok && sched.item(cl, j, t, kb0, kb1); ++j) {
        const int acc = j % Cfg::NBUF;
        const uint32_t use = (uint32_t)(j / Cfg::NBUF);
        const uint32_t d_tmem = tmem_base + (uint32_t)(acc * Cfg::TILE_N);
        int kb = kb0;
        bool tl_first = true;
        if constexpr (NT == 2) {
          // One accumulator of two 256-column regions, released region by region by the epilogue
          // (tempty_bar(0) / tempty_bar(1)): while region 1 of the previous tile still drains,
          // the first STAGES k-blocks already accumulate into region 0; their slots are freed only
          // once region 1 has consumed them too.
          if (!wait_tempty(0, (use & 1u) ^ 1u)) { ok = false; break; }
          const int pre = min(Cfg::STAGES, kb1 - kb0);
          const int s0 = stage;
          const uint32_t p0 = phase;
          for (int i = 0; i < pre; ++i) {
            if (!wait_full(stage, phase)) { ok = false; break; }
            if (tl && lane == 0 && i == 0 && j < 8) { tl[4 * j] = globaltimer_ns(); tl_first = false; }
            issue(d_tmem, stage, i == 0, 0, 1);
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
          }
          if (!ok || !wait_tempty(1, (use & 1u) ^ 1u)) { ok = false; break; }
          stage = s0;
          phase = p0;
          for (int i = 0; i < pre; ++i) {
            issue(d_tmem, stage, i == 0, 1, 2);
            tc_commit_warp<CG>(empty_bar(stage), MC == 2 ? (uint16_t)0xF : (uint16_t)0x3);
            __syncwarp();
            if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
          }
          kb = kb0 + pre;
        } else {
          if (!wait_tempty(acc, (use & 1u) ^ 1u)) { ok = false; break; }
          // (MM_EXP bit 0: the previous tile's read-out finishes before this tile's MMAs start)
          if ((args.exp & 1) && j > 0 && !wait_tempty(acc ^ 1, ((uint32_t)((j - 1) / 2) & 1u))) { ok = false; break; }
        }
        const bool half_item = NT == 1 && CG == 2 && MC == 1 && sched.half_of(cl, j) >= 0;
        for (; kb < kb1; ++kb) {
          if (!wait_full(stage, phase)) { ok = false; break; }
          if (tl && lane == 0 && tl_first && j < 8) { tl[4 * j] = globaltimer_ns(); tl_first = false; }
          if (half_item) issue_half(d_tmem, stage, kb == kb0);
          else issue(d_tmem, stage, kb == kb0, 0, NT);
          // frees this smem stage when the MMAs retire: in both CTAs of the pair, and with MC = 2 also
          // in the other pair, whose producers multicast into this pair's slots
          tc_commit_warp<CG>(empty_bar(stage), MC == 2 ? (uint16_t)0xF : (uint16_t)0x3);
          __syncwarp();
          if (++stage == Cfg::STAGES) { stage = 0; phase ^= 1u; }
        }
        if (!ok) break;
        if (tl && lane == 0 && j < 8) tl[4 * j + 1] = globaltimer_ns();
        tc_commit_warp<CG>(tfull_bar(acc), (uint16_t)(0x3u << leader));  // accumulator ready (both CTAs)
        __syncwarp();
      }
    }
  } else {
    // ---------------------------------------------------------------- epilogue (warps 2..9)
    // Eight warps: two per TMEM lane quarter q (warp w may only read lanes 32*(w%4)..+31) taking
    // alternate 32-column chunks (h = 0 the even ones, h = 1 the odd ones) in column order, so for
    // NT=2 all eight drain region 0 first and release it halfway through the read-out.
    const uint32_t ew = warp - 2;           // epilogue warp 0..7
    const uint32_t q = warp & 3u;           // TMEM lane quarter
    const int h = (int)(ew >> 2);           // column half
    uint32_t* C = reinterpret_cast<uint32_t*>(args.C);
    uint32_t* part = reinterpret_cast<uint32_t*>(args.ws);
    const bool vec_ok = ((args.ldc & 3) == 0) && ((reinterpret_cast<uintptr_t>(args.C) & 15) == 0);
    const int prow = (int)(q * 32 + lane);  // row of this thread inside the CTA's 128-row slab
    constexpr int NCH = Cfg::TILE_N / 32;   // 32-column chunks per accumulator
    constexpr int HCH = NCH / 2;            // chunks per warp: c(i) = h + 2 i
    // C chunk (32 rows x 32 columns) -> global: through this warp's 128B-swizzled 4-KB smem buffer
    // and one TMA store (full lines, edges clipped by the tensor map), or, when C's base/pitch rule
    // out TMA, straight from registers with predicated stores.
    const uint32_t ebuf = sEpi + ew * 4096u;
    uint32_t n_stores = 0;
    auto emit = [&](const uint32_t (&v)[32], int64_t row_base, int64_t col0, bool red = false) {
      if (I8 && args.res_m) {  // (compiled into the INT8 kernels only)
        const int bb = args.bat_rows ? (int)(row_base / args.bat_rows) : 0;
        const int rm = args.res_mt[bb], rc16 = args.res_c16t[bb];
        const float rrcp = args.res_rcpt[bb];
        // MM_F64_EMU: the exact INT32 values reduced mod res_m to bytes — x = 2^16 h + l, y = h·(2^16
        // mod m) + l ≡ x (|y| < 2^24, exact in float), r = y − m·floor(y/m) corrected — 32 bytes per
        // row, staged unswizzled (32 rows × 32 B) and stored by one TMA store (uint8 map, no reduce-add)
        uint32_t w[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          uint32_t word = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int x = (int)v[4 * i + u];
            const int y = (x >> 16) * rc16 + (x & 0xFFFF);
            int r = y - __float2int_rd(__int2float_rn(y) * rrcp) * rm;
            r += r < 0 ? rm : 0;
            r -= r >= rm ? rm : 0;
            word |= (uint32_t)r << (8 * u);
          }
          w[i] = word;
        }
        if (n_stores >= 1) {
          if (lane == 0) bulk_wait_read<0>();
          __syncwarp();
        }
        st_shared_v4(ebuf + lane * 32u, w[0], w[1], w[2], w[3]);
        st_shared_v4(ebuf + lane * 32u + 16u, w[4], w[5], w[6], w[7]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_2d(&tmC, ebuf, (int32_t)col0, (int32_t)row_base);
          bulk_commit();
        }
        ++n_stores;
        return;
      }
      if (args.c_tma) {
        const uint64_t c0 = args.trace ? clock64() : 0;
        if (n_stores >= 1) {
          if (lane == 0) bulk_wait_read<0>();  // this warp's previous store has read the buffer
          __syncwarp();
        }
        const uint64_t c1 = args.trace ? clock64() : 0;
#pragma unroll
        for (int i = 0; i < 8; ++i)
          st_shared_v4(ebuf + lane * 128u + ((uint32_t)(i ^ (int)(lane & 7u)) << 4), v[4 * i], v[4 * i + 1],
                       v[4 * i + 2], v[4 * i + 3]);
        const uint64_t c2 = args.trace ? clock64() : 0;
        if (!(args.debug & 8)) fence_proxy_async_smem();  // (diagnostics: bit 3 skips the fence)
        __syncwarp();
        const uint64_t c3 = args.trace ? clock64() : 0;
        if (lane == 0 && !(args.debug & 4)) {  // (diagnostics: bit 2 skips the store)
          if (red) tma_reduce_add_2d(&tmC, ebuf, (int32_t)col0, (int32_t)row_base);
          else tma_store_2d(&tmC, ebuf, (int32_t)col0, (int32_t)row_base);
          bulk_commit();
        }
        if (args.trace) {
          tr_c[3] += (c1 - c0) + (clock64() - c3);
          tr_c[1] += c2 - c1;
          tr_c[2] += c3 - c2;
          tr_c[4] += 1;
        }
        ++n_stores;
      } else {
        store_row32(C, args.ldc, row_base + lane, col0, args.M, args.N, v, vec_ok);
      }
    };
    // TMEM accumulator (NT=1) or region (NT=2) a has been read out by this warp: let the MMA warp
    // reuse it once all eight have
    auto release = [&](int a) {
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (CG == 2) mbar_arrive_cluster(mapa_shared(tempty_bar(a), leader));
        else mbar_arrive(tempty_bar(a));
      }
    };
    // Split tiles (sched.cuh): no CTA ever waits for one that may not have started.  Each part
    // of a split tile takes a ticket (one atomic per CTA, shared with the eight epilogue warps);
    // only a CTA that holds a ticket waits, and only for parts whose tickets were taken earlier —
    // CTAs already running whose remaining work (zeroing, or publishing a partial slab) waits on
    // nothing.  Counters: tickets [0, T·CG·MC), publish counts [T·CG·MC, 2·T·CG·MC).
    const size_t tcount = (size_t)sched.tiles_m * sched.tiles_n * (CG * MC);
    auto take_ticket = [&](unsigned* ctr) -> unsigned {
      if (ew == 0 && lane == 0) *tick_slot = atomic_add_acq_rel_gpu(ctr, 1u);
      asm volatile("bar.sync 1, 256;" ::: "memory");
      const unsigned tk = *tick_slot;
      asm volatile("bar.sync 1, 256;" ::: "memory");
      return tk;
    };
    // partial slab of cluster cc for a split tile whose first part is held by c_first: each cluster
    // has at most two split parts (the first and the last segment of its tail range), one slot each
    auto slab_of = [&](int cc, int c_first) {
      const size_t role = cc == c_first ? 1 : 0;
      return reinterpret_cast<uint4*>(part + (((size_t)cc * 2 + role) * (CG * MC) + crank) * (128 * Cfg::TILE_N));
    };
    int t, kb0, kb1;
    for (int j = 0; sched.item(cl, j, t, kb0, kb1); ++j) {
      int tm, tn;
      sched.tile_coords(t, tm, tn);
      const int acc = j % Cfg::NBUF;
      const uint32_t use = (uint32_t)(j / Cfg::NBUF);
      // reduce-add tail (sched.red): both halves add into C with TMA reduce-add; the half that takes
      // the first ticket zeroes this CTA's rows of the tile in C while its MMAs run and publishes it
      const bool red_item = sched.red && !(kb0 == 0 && kb1 == num_kb);
      unsigned* red_flag = args.flags + (size_t)t * (CG * MC) + crank;
      bool red_zeroer = false;
      if (red_item) {
        // the ticket and the zeros follow no load of this launch: wait for the previous kernel in the
        // stream (PDL) first, or the zeros could land before that kernel's own stores to the same C
        pdl_wait();
        red_zeroer = take_ticket(red_flag) == 0u;
      }
      if (red_zeroer) {
        const int64_t zrow = (int64_t)tm * Cfg::M_TILE + pair * Cfg::M_MMA + rank * Cfg::BM + q * 32;
        if (n_stores >= 1) {
          if (lane == 0) bulk_wait_read<0>();  // this warp's previous store has read the buffer
          __syncwarp();
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) st_shared_v4(ebuf + lane * 128u + (uint32_t)i * 16u, 0u, 0u, 0u, 0u);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          for (int c = h; c < NCH; c += 2) tma_store_2d(&tmC, ebuf, (int32_t)((int64_t)tn * Cfg::TILE_N + c * 32), (int32_t)zrow);
          bulk_commit();
          bulk_wait<0>();  // the zeros are in global memory
        }
        ++n_stores;
        __syncwarp();
        asm volatile("bar.sync 1, 256;" ::: "memory");
        if (ew == 0 && lane == 0) {
          asm volatile("fence.proxy.async.global;" ::: "memory");  // async-proxy writes before the release
          red_release_gpu_add(red_flag, 2u);  // ticket (1) + ticket (1) + zeroed (2) = 4
        }
      }
      const uint64_t tq0 = args.trace ? globaltimer_ns() : 0;
      if (!mbar_wait(tfull_bar(acc), use & 1u, err, 4)) break;
      if (args.trace) tr_tfull += globaltimer_ns() - tq0;
      const uint64_t td0 = args.trace ? globaltimer_ns() : 0;  // accumulator read-out time
      if (tl && ew == 0 && lane == 0 && j < 8) tl[4 * j + 2] = td0;
      tc_fence_after();
      const int64_t row = (int64_t)tm * Cfg::M_TILE + pair * Cfg::M_MMA + rank * Cfg::BM + prow;
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + (uint32_t)(acc * Cfg::TILE_N);
      const bool whole = (kb0 == 0 && kb1 == num_kb);
      const int tail_c = cl;  // tail items: cluster index == tail-slot index
      const int64_t row_base = row - lane;  // first row of this warp's 32-row block
      const int64_t col_t = (int64_t)tn * Cfg::TILE_N;
      if (red_item) {
        if (!red_zeroer) {
          // wait until the other half (it took the first ticket, so it is running) has zeroed these
          // rows, then reset the counter for the next launch
          if (ew == 0 && lane == 0) {
            if (counter_wait(red_flag, 4u, err, 8)) *(volatile unsigned*)red_flag = 0u;
            asm volatile("fence.proxy.async.global;" ::: "memory");  // acquired zeros before the reduce-adds
          }
          __syncwarp();
          asm volatile("bar.sync 1, 256;" ::: "memory");
        }
#pragma unroll 1
        for (int c = h; c < NCH; c += 2) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + c * 32, v);
          tmem_ld_wait();
          emit(v, row_base, col_t + c * 32, true);
        }
      } else if (NT == 1 && sched.half_of(cl, j) >= 0) {
        // N-half tail item: 128 columns (chunks 0..3) starting at the half's first column
        const int64_t col_h = col_t + (int64_t)sched.half_of(cl, j) * (kBN / 2);
#pragma unroll 1
        for (int c = h; c < NCH / 2; c += 2) {
          uint32_t v[32];
          tmem_ld_32x32b_x32(t_row + c * 32, v);
          tmem_ld_wait();
          emit(v, row_base, col_h + c * 32);
        }
      } else if (whole) {
        // software-pipelined: the TMEM load of chunk c+1 is in flight while chunk c is stored
        uint32_t va[32], vb[32];
        tmem_ld_32x32b_x32(t_row + h * 32, va);
        tmem_ld_wait();
#pragma unroll 1
        for (int i = 0; i < HCH; i += 2) {
          const int c = h + 2 * i;  // chunks c and c + 2
          tmem_ld_32x32b_x32(t_row + (c + 2) * 32, vb);
          emit(va, row_base, col_t + c * 32);
          const uint64_t w0 = args.trace ? clock64() : 0;
          tmem_ld_wait();
          if (args.trace) tr_c[0] += clock64() - w0;
          if (i + 2 < HCH) tmem_ld_32x32b_x32(t_row + (c + 4) * 32, va);
          emit(vb, row_base, col_t + (c + 2) * 32);
          tmem_ld_wait();
          if (NT == 2 && i + 2 == HCH / 2) release(0);  // region 0 (chunks 0..7) read out: its MMAs may start
        }
      } else {
        // Split tile (modes 1, 2): segments c_first .. c_last of the tail range hold its k-blocks in
        // order (c_first from k-block 0).  Every part but the last to finish publishes its slab; the
        // last adds all of them in segment order — the same fixed order whoever finishes last, so
        // results are run-to-run identical.
        const int64_t ti0 = (int64_t)(t - sched.W * sched.nc) * num_kb;
        const int c_first = sched.tail_cluster_of(ti0);
        const int c_last = sched.tail_cluster_of(ti0 + num_kb - 1);
        const unsigned nparts = (unsigned)(c_last - c_first + 1);
        unsigned* tick = args.flags + (size_t)t * (CG * MC) + crank;
        unsigned* pub = tick + tcount;
        if (take_ticket(tick) + 1u < nparts) {
          uint4* slot = slab_of(tail_c, c_first);
#pragma unroll 1
          for (int c = h; c < NCH; c += 2) {
            uint32_t v[32];
            tmem_ld_32x32b_x32(t_row + c * 32, v);
            tmem_ld_wait();
#pragma unroll
            for (int i = 0; i < 8; ++i)
              st_cg_u4(slot + slab_index(c, (int)q, i, (int)lane), make_uint4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]));
          }
          __threadfence();
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (ew == 0 && lane == 0) red_release_gpu_add(pub, 1u);
        } else {
          // last part: the others took their tickets earlier, so they are running and only publishing
          if (ew == 0 && lane == 0) {
            if (counter_wait(pub, nparts - 1u, err, 6)) {
              *(volatile unsigned*)tick = 0u;  // reset both counters for the next launch
              *(volatile unsigned*)pub = 0u;
            }
          }
          __syncwarp();  // reconverge warp 2 before the (.aligned) named barrier
          asm volatile("bar.sync 1, 256;" ::: "memory");
          if (sched.land && nparts == 2u) {
            // Exact-halves split: this is the cluster's last item, so its operand ring is idle (all
            // loads consumed, all MMAs retired).  Land the other half's slab there with one 4-KB bulk
            // copy per chunk (all in flight at once), then add it from shared memory (two FP32 addends
            // commute exactly, so the order of the halves does not matter).
            const int other = tail_c == c_first ? c_last : c_first;
            const uint8_t* src = reinterpret_cast<const uint8_t*>(slab_of(other, c_first));
            if (lane == 0) {
              // the slab was written by another SM through the generic proxy and acquired above;
              // order that before the async-proxy (bulk copy) reads of it
              asm volatile("fence.proxy.async.global;" ::: "memory");
              mbar_arrive_expect_tx(land_bar((int)ew), HCH * 4096u);
              for (int c = h; c < NCH; c += 2)
                bulk_copy_g2s(sA + (uint32_t)(c * 4 + q) * 4096u, src + slab_index(c, (int)q, 0, 0) * 16, 4096u,
                              land_bar((int)ew));
            }
            mbar_wait(land_bar((int)ew), 0u, err, 7);
#pragma unroll 1
            for (int c = h; c < NCH; c += 2) {
              uint32_t v[32];
              tmem_ld_32x32b_x32(t_row + c * 32, v);
              uint4 w[8];
#pragma unroll
              for (int i = 0; i < 8; ++i)
                w[i] = *reinterpret_cast<const uint4*>(smem + (size_t)(c * 4 + q) * 4096 + i * 512 + lane * 16);
              tmem_ld_wait();
              add_words<I8>(v, w);
              emit(v, row_base, col_t + c * 32);
            }
          } else {
#pragma unroll 1
            for (int c = h; c < NCH; c += 2) {
              uint32_t o[32], v[32];
              tmem_ld_32x32b_x32(t_row + c * 32, o);
              tmem_ld_wait();
              // v = part(c_first) + part(c_first+1) + ... + part(c_last), this CTA's own from TMEM
              if (c_first == tail_c) {
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = o[i];
              } else {
                const uint4* s0 = slab_of(c_first, c_first) + slab_index(c, (int)q, 0, (int)lane);
#pragma unroll
                for (int i = 0; i < 8; ++i) {
                  const uint4 w = ld_cg_u4(s0 + i * 32);
                  v[4 * i] = w.x; v[4 * i + 1] = w.y; v[4 * i + 2] = w.z; v[4 * i + 3] = w.w;
                }
              }
              for (int qq = c_first + 1; qq <= c_last; ++qq) {
                if (qq == tail_c) add_regs<I8>(v, o);
                else add32<I8>(v, slab_of(qq, c_first) + slab_index(c, (int)q, 0, (int)lane));
              }
              emit(v, row_base, col_t + c * 32);
            }
          }
        }
      }
      if (NT == 2) {
        if (!whole) release(0);
        release(1);
      } else {
        release(acc);
      }
      if (args.trace) tr_drain += globaltimer_ns() - td0;
      if (tl && ew == 0 && lane == 0 && j < 8) tl[4 * j + 3] = globaltimer_ns();
    }
    if (args.c_tma && lane == 0) bulk_wait<0>();  // all output stores complete before exit
  }

  __syncwarp();
  tc_fence_before();
  if constexpr (CG == 2) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (warp == 1) tmem_dealloc<CG>(tmem_base, 512);
  if (args.trace) {
    unsigned long long* tr = args.trace + (size_t)blockIdx.x * 16;
    if (warp == 0 && lane == 0) { tr[0] = tr_barrier; tr[1] = tr_empty; }
    if (warp == 1 && lane == 0) {
      tr[2] = tr_tempty; tr[3] = tr_full; tr[6] = tr_t0; tr[7] = globaltimer_ns();
      tr[13] = clock64() - tr_clk0;  // SM cycles over the CTA's life: effective clock = tr[13] / (tr[7] - tr[6])
      tr[14] = tr_entry;
    }
    if (warp == 2 && lane == 0) {
      tr[4] = tr_tfull;
      tr[5] = tr_drain;
      for (int k = 0; k < 5; ++k) tr[8 + k] = tr_c[k];
    }
  }
  if (args.clk && threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long* r = args.clk + 4 * (size_t)blockIdx.x;
    r[0] = clk_c0;
    r[1] = clk_t0;
    r[2] = clock64();
    r[3] = globaltimer_ns();
  }
  // the last CTA to finish resets the wave-barrier counters (and the abandoned flag) for the next launch
  if (args.wave_sync && threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(args.sync + 1, 1u) == gridDim.x - 1) {
      atomicExch(args.sync, 0u);
      atomicExch(args.sync + 2, 0u);
      atomicExch(args.sync + 1, 0u);
    }
  }
}

// max_clusters: how many clusters of cg*mc CTAs can be co-resident (the persistent grid and the
// wave barrier need all of them resident at once); <= 0: num_sms / (cg*mc).
WorkSched make_sched(bool i8, int cg, int nt, int mc, int64_t M, int64_t N, int64_t K, int num_sms, int max_clusters,
                     int ka = 1, bool c_tma = true) {
  const int m_mma = 128 * cg * mc;
  const int bk = (i8 ? 128 : 64) * ka;
  const int tiles_m = (int)((M + m_mma - 1) / m_mma);
  const int tiles_n = (int)((N + kBN * nt - 1) / (kBN * nt));
  // measured best (tools/sweep_raster.py): 256-wide tiles 8 tile-rows x ~9 tile-cols per 74-cluster wave;
  // 512-wide tiles 16 x ~4.6
  int group_m = (nt == 2 ? 16 : 8) / mc;
  const int num_kb = (int)((K + bk - 1) / bk);
  const int64_t T = (int64_t)tiles_m * tiles_n;
  int64_t nc = num_sms / (cg * mc);
  if (max_clusters > 0) nc = std::min<int64_t>(nc, max_clusters);
  nc = std::max<int64_t>(1, std::min<int64_t>(nc, T * 4));  // at most ~4 clusters share one tile
  // INT8, 256-wide tiles, at most 4 waves: groups of 4 tile-rows (measured: 3072^3 +6.8 %,
  // C3 4096^3 +3.5 %; 6144^3 / 8192^3 -1.3 / -1.8 % and BF16 neutral, so only there)
  if (i8 && nt == 1 && mc == 1 && T <= 4 * nc) group_m = 4;
  if (const char* e = knob("MM_GROUP_M")) group_m = atoi(e) > 0 ? atoi(e) : group_m;  // tuning knob
  const int64_t tail = T % nc;
  // The split tail pays for its partial-slab round trip only when there are many full waves
  // (measured: C4 55 waves +0.6 %, C3 3 waves -12 %; tools/ab_gpu.py).
  // Default: split the tail tiles into exact halves when there are enough clusters
  // (2*tail <= nc) and 256-wide tiles (a 128 x 256 slab fits the idle operand ring of the
  // half that finishes last, which then lands the other's slab with bulk copies); MM_STREAMK=1 forces
  // the general split (partials read from global memory), MM_STREAMK=0 disables both.
  // (bf16 only: int8 tiles are half as long, so the fixed fix-up cost outweighs the saved
  // half tile — measured C3 -3.4 %, bf16 4096^3 +4.1 %, tools/ab_gpu.py)
  // Mode 3 (when C takes TMA stores): the same exact halves, both added into C (zeroed by
  // the half that takes the first ticket, while its MMAs run) with TMA reduce-add stores —
  // no partial slabs, no read-back, neither half waits for the other's MMAs.
  // Reduce-add stores take ~1.5x as long as plain ones and the zeroing half stores the tile twice,
  // so int8 (half-length tiles) gains only with long K (C3 K=4096: neutral; 2560^3 -7 %),
  // bf16 4096^3 +4 %, 2560^3 +5 % over landing (tools/ab_gpu.py).
  int mode = 0;
  // (the zeroing and the slower reduce-add read-out cost a few us: the saved half tile must be
  // longer — K >= 2304 (BF16: 1536 -4..-6 %, 2048 0..-4 %, 2304 +5.5 %, 3072 +9.5 %) / 4608
  // (INT8: 4096 neutral, 5120 +2 %, 5632 +5 %); a single 256^3 tile split in halves ran
  // 8.2 -> 10.8 us)
  if (tail > 0 && mc == 1 && 2 * tail <= nc && K >= (i8 ? 4608 : 2304))
    mode = c_tma ? 3 : ((!i8 && nt == 1 && num_kb >= 8) ? 2 : 0);
  // Round 2: the tail tiles of 256-wide pair tiles as two N halves on two clusters (pair MMA N = 128,
  // whole K each): no partial sums and no reduce-add, so it beats whole tiles at every K and the K
  // halves below K = 3072 (BF16) / 6144 (INT8) — measured at 4096 x K x 4096 (34-tile tail):
  // INT8 K = 2048 / 3072 / 4096 / 5120: 0.0389 / 0.0482 / 0.0584 / 0.0702 ms vs K halves 0.0461 /
  // 0.0543 / 0.0615 / 0.0707 and whole tiles 0.0399 / 0.0502 / 0.0604 / 0.0707; BF16 K = 768 / 1536
  // / 2048 / 2560: 33.8 / 50.2 / 62.5 / 72.7 us vs 42.0 / 56.4 / 64.5 / 74.8 (K halves); from
  // BF16 K = 4096 / INT8 K = 8192 the K halves win (profiles/sweep_tail_r2o.txt).  Without a
  // reduce-add (C not TMA-storable, or in a peer's memory) N halves replace the landing split.
  if (tail > 0 && mc == 1 && cg == 2 && nt == 1 && 2 * tail <= nc &&
      (K < (i8 ? 6144 : 3072) || !c_tma))
    mode = 4;
  if (const char* e = knob("MM_STREAMK")) mode = tail > 0 ? atoi(e) : 0;  // tuning knob
  if (mode == 4 && (nt != 1 || cg != 2 || mc != 1 || 2 * tail > nc)) mode = 0;  // N halves: 256-wide pair tiles
  if (knob("MM_ONE_TILE")) return sched_build(tiles_m, tiles_n, group_m, num_kb, (int)T, 0);  // (A/B knob: one tile per cluster, non-persistent)
  if (mc != 1) mode = 0;                // (cluster-pair multicast: whole tiles only)
  if (mode == 2 && (nt != 1 || 2 * tail > nc)) mode = 1;  // landing: 256-wide tiles, one partner per tile
  if (mode == 3 && (!c_tma || 2 * tail > nc)) mode = 1;
  return sched_build(tiles_m, tiles_n, group_m, num_kb, (int)nc, mode);
}

template <bool I8, int CG, int NT, int MC, int KA = 1>
cudaError_t launch_cfg(cudaLaunchConfig_t& cfg, cudaLaunchAttribute* attr, int num_sms, int* max_clusters) {
  using Cfg = TcCfg<I8, CG, NT, MC, KA>;
  auto kern = gemm_tc_kernel<I8, CG, NT, MC, KA>;
  // per template instance and device (function attributes and occupancy are per device)
  static std::atomic<int> max_cl_dev[kMaxDevices];  // 0 = not set up yet, -1 = query failed
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  cfg = {};
  cfg.blockDim = dim3(kThreads, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = CG * MC;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  attr[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;  // (the occupancy query below: cluster shape only)
  int max_cl = max_cl_dev[dev].load();
  if (max_cl == 0) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    // all clusters of the persistent grid must be resident together (wave barrier, stream-K waits)
    cfg.gridDim = dim3((unsigned)(num_sms / (CG * MC) * CG * MC), 1, 1);
    int n = 0;
    if (cudaOccupancyMaxActiveClusters(&n, (void*)kern, &cfg) != cudaSuccess) {
      cudaGetLastError();
      n = 0;
    }
    max_cl = n > 0 ? n : -1;
    max_cl_dev[dev].store(max_cl);
  }
  *max_clusters = max_cl > 0 ? max_cl : 0;
  cfg.numAttrs = knob("MM_NO_PDL") ? 1 : 2;  // + programmatic dependent launch (knob: MM_NO_PDL=1 off)
  return cudaSuccess;
}

template <bool I8, int CG, int NT, int MC, int KA = 1>
cudaError_t launch_impl(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmC, const CUtensorMap& tmBh,
                        const GemmArgs& a, int num_sms, cudaStream_t s) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[2];
  int max_cl = 0;
  cudaError_t e = launch_cfg<I8, CG, NT, MC, KA>(cfg, attr, num_sms, &max_cl);
  if (e != cudaSuccess) return e;
  const WorkSched sched = make_sched(I8, CG, NT, MC, a.M, a.N, a.K, num_sms, max_cl, KA, a.c_tma != 0 && !a.no_reduce);
  cfg.gridDim = dim3(sched.nc * CG * MC, 1, 1);
  cfg.stream = s;
  return cudaLaunchKernelEx(&cfg, gemm_tc_kernel<I8, CG, NT, MC, KA>, tmA, tmB, tmC, tmBh, a, sched);
}

template <bool I8, int CG, int NT, int MC, int KA = 1>
int max_clusters_of(int num_sms) {
  cudaLaunchConfig_t cfg;
  cudaLaunchAttribute attr[2];
  int max_cl = 0;
  if (launch_cfg<I8, CG, NT, MC, KA>(cfg, attr, num_sms, &max_cl) != cudaSuccess) return 0;
  return max_cl;
}

int max_clusters_impl(bool i8, int cg, int nt, int mc, int ka, int num_sms) {
  if (cg == 1) return i8 ? max_clusters_of<true, 1, 1, 1>(num_sms) : max_clusters_of<false, 1, 1, 1>(num_sms);
  if (nt == 1 && ka == 2) {
    if (mc == 2) return i8 ? max_clusters_of<true, 2, 1, 2, 2>(num_sms) : max_clusters_of<false, 2, 1, 2, 2>(num_sms);
    return i8 ? max_clusters_of<true, 2, 1, 1, 2>(num_sms) : max_clusters_of<false, 2, 1, 1, 2>(num_sms);
  }
  if (mc == 2) {
    if (i8) return nt == 2 ? max_clusters_of<true, 2, 2, 2>(num_sms) : max_clusters_of<true, 2, 1, 2>(num_sms);
    return nt == 2 ? max_clusters_of<false, 2, 2, 2>(num_sms) : max_clusters_of<false, 2, 1, 2>(num_sms);
  }
  if (i8) return nt == 2 ? max_clusters_of<true, 2, 2, 1>(num_sms) : max_clusters_of<true, 2, 1, 1>(num_sms);
  return nt == 2 ? max_clusters_of<false, 2, 2, 1>(num_sms) : max_clusters_of<false, 2, 1, 1>(num_sms);
}

}  // namespace

int max_clusters(bool i8, int cg, int nt, int mc, int ka, int num_sms) { return max_clusters_impl(i8, cg, nt, mc, ka, num_sms); }

void tc_box_dims(bool i8, int cg, int mc, int ka, uint32_t* a_box, uint32_t* b_box) {
  const uint32_t esz = i8 ? 1 : 2;
  a_box[0] = 128 / esz;       // K elements (128 B)
  a_box[1] = 128;             // rows
  b_box[0] = 128 / esz;       // N elements (128 B)
  b_box[1] = 128 / esz * ka / mc;  // K rows (BK, or the half of it one pair loads when two pairs share B)
  (void)cg;
}

void tc_plan_needs(bool i8, int cg, int nt, int mc, int ka, int64_t M, int64_t N, int64_t K, int num_sms,
                   size_t* ws_bytes, size_t* flag_count) {
  const int mcl = max_clusters_impl(i8, cg, nt, mc, ka, num_sms);
  const WorkSched sc = make_sched(i8, cg, nt, mc, M, N, K, num_sms, mcl, ka, true);
  const WorkSched sc2 = make_sched(i8, cg, nt, mc, M, N, K, num_sms, mcl, ka, false);  // (C without TMA stores)
  // two partial-slab slots per cluster (its first and its last tail segment), tickets + publish counts
  *ws_bytes = (size_t)std::max(sc.ntc, sc2.ntc) * 2 * cg * mc * 128 * kBN * nt * 4;
  *flag_count = (size_t)sc.tiles_m * sc.tiles_n * cg * mc * 2;
}

cudaError_t launch_gemm_tc(bool i8, int cg, int nt, int mc, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmC, const CUtensorMap& tmBh, const GemmArgs& a, int num_sms,
                           cudaStream_t s) {
  if (cg == 1)
    return i8 ? launch_impl<true, 1, 1, 1>(tmA, tmB, tmC, tmBh, a, num_sms, s)
              : launch_impl<false, 1, 1, 1>(tmA, tmB, tmC, tmBh, a, num_sms, s);
  if (mc == 2 && nt == 1 && a.ka == 2)
    return i8 ? launch_impl<true, 2, 1, 2, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s)
              : launch_impl<false, 2, 1, 2, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s);
  if (mc == 2) {
    if (i8)
      return nt == 2 ? launch_impl<true, 2, 2, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s)
                     : launch_impl<true, 2, 1, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s);
    return nt == 2 ? launch_impl<false, 2, 2, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s)
                   : launch_impl<false, 2, 1, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s);
  }
  if (nt == 1 && a.ka == 2)
    return i8 ? launch_impl<true, 2, 1, 1, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s)
              : launch_impl<false, 2, 1, 1, 2>(tmA, tmB, tmC, tmBh, a, num_sms, s);
  if (i8)
    return nt == 2 ? launch_impl<true, 2, 2, 1>(tmA, tmB, tmC, tmBh, a, num_sms, s)
                   : launch_impl<true, 2, 1, 1>(tmA, tmB, tmC, tmBh, a, num_sms, s);
  return nt == 2 ? launch_impl<false, 2, 2, 1>(tmA, tmB, tmC, tmBh, a, num_sms, s)
                 : launch_impl<false, 2, 1, 1>(tmA, tmB, tmC, tmBh, a, num_sms, s);
}

}  // namespace mmb
