// gemm_f64.cu — C (+)= A·B in IEEE binary64, the paper's own precision
// (`double`), on the FP64 tensor pipe.
//
// sm_100a has no FP64 tcgen05 kind, so the MMA is the warp-level
// mma.sync.m8n8k4.f64 (SASS DMMA.8x8x4) with register accumulators; the
// operand pipeline is still Blackwell-native: TMA 2-D boxes into a
// 128-byte-swizzled shared-memory ring with full/empty mbarriers between one
// producer warp and the consumer warps ("cache tiling",
// PAPER.md:366-373 prefetching/pipelining, done by TMA instead of the CPU).
//
// Work split (sched.cuh): whole tiles in grouped-raster waves over the persistent
// CTAs (concurrent tiles share A row panels and B column panels in L2), then the
// tiles of the last, partial wave split "stream-K" style over all CTAs, so every
// SM gets the same number of DMMA k-blocks (C2: 224 tiles on 148 SMs = 1 wave +
// an even tail).  The parts of a split tile take tickets; all but the last to finish
// publish partial tiles to a workspace, and the last adds them in segment order — a
// fixed order, so results are run-to-run identical — without any CTA waiting for one
// that may not be resident yet.
//
// CTA tile BM×BN (128×128; 64×64 or 32×32 for small problems, where 32×32 tiles
// give every CTA one whole tile and no fix-up: C1 = 64 tiles), K slab 16 (one
// 128-B swizzle row of A).  WM×WN consumer warps, each owning a (BM/WM)×(BN/WN)
// sub-tile: 16 warps (4 per SM sub-partition) at 128×128 and 64×64, so a warp
// stalled at a k-block boundary leaves three to keep the DMMA pipe busy.
// Fragment loads are conflict-free with the swizzle because each DMMA's four
// k indices are taken from rows {b, b+1, b+4, b+5} of the slab (b ∈ {0,2,8,10}):
// the same four k's for A and B, so each DMMA still adds A[i][k]·B[k][j] over
// its four k's; only which k's are grouped together changes.
// Edges: TMA zero-fills out-of-bounds reads; stores are predicated.
#include <atomic>

#include "kernels.h"
#include "knobs.h"
#include "ptx.cuh"
#include "sched.cuh"

namespace mmb {

namespace {

constexpr int BK = 16;
constexpr int BBOX_BYTES = BK * 16 * 8;  // 2 KB, box {16 cols, 16 rows}

// KS: k-block groups of WM x WN consumer warps.  KS = 2 (small tiles): the two groups take the
// even / odd k-blocks of each tile (twice the DMMA chains in flight per SMSP), and group 1's
// accumulators are added into group 0's through shared memory before the epilogue.
// KB: k-blocks per TMA load (small tiles: one 3-D box of A and one of B bring KB consecutive
// k-blocks into KB consecutive ring slots, so a 32x32 tile's whole K arrives in a few loads — a
// single thread issuing three 2-D loads per 16-deep k-block was the bottleneck at C1: ~160
// cycles per load).  B then sits per group as [column box][KB x 16 rows][128 B].
// CK: CTAs per tile along K (a cluster of CK CTAs on CK SMs; CK = 2 for problems with at most half
// a wave of 32x32 tiles, e.g. C1: 64 tiles on 128 SMs instead of 64).  Rank 1 adds nothing itself:
// it stores its partial tile into rank 0's shared memory (distributed shared memory) and arrives on
// rank 0's exchange barrier; rank 0 adds it to its own (fixed order) and writes C.
template <int BM, int BN, int WM, int WN, int KS = 1, int KB = 1, int CK = 1>
struct F64Cfg {
  static constexpr int NTILE = WM * WN;        // warps covering one tile
  static constexpr int NCONS = NTILE * KS;     // consumer warps
  static constexpr int THREADS = (NCONS + 1) * 32;
  static constexpr int A_BYTES = BM * BK * 8;  // one box {16, BM}
  static constexpr int NBBOX = BN / 16;
  static constexpr int B_BYTES = NBBOX * BBOX_BYTES;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  // ~200 KB of operand ring: 6 stages at 128x128, 12 at 64x64, 25 at 32x32 (a whole K <= 384 of a
  // small tile in flight at once: the cold DRAM round trip is paid once, not K/(16*stages) times)
  static constexpr int SCR_BYTES = (KS - 1) * BM * BN * 8;  // accumulators of groups 1..KS-1
  static constexpr int XSCR_BYTES = (CK - 1) * BM * BN * 8;  // rank 0: the other K half's partial tile
  // (and never more than the 227 KB a CTA may hold with the scratch: KS = 8 has 56 KB of it)
  static constexpr int RING_MAX = 225 * 1024 - 2048 - SCR_BYTES - XSCR_BYTES;
  static constexpr int RING = (200 * 1024) < RING_MAX ? (200 * 1024) : RING_MAX;
  static constexpr int STAGES0 = RING / STAGE_BYTES < 64 ? RING / STAGE_BYTES : 64;
  static constexpr int STAGES = STAGES0 / KB * KB;            // whole groups of KB slots
  static constexpr int BOX_STRIDE = KB * BBOX_BYTES;          // between B column boxes of one slot
  static constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 1024 + SCR_BYTES + XSCR_BYTES + 1024;
  static_assert(STAGES >= 4 && 16 * STAGES <= 1008, "ring (+ the ticket word at the end of the barrier area)");
  static constexpr int MI = BM / WM / 8;  // 8-row DMMA tiles per warp
  static constexpr int NI = BN / WN / 8;  // 8-col DMMA tiles per warp (even: pairs share a 16-col box)
  static_assert(NI % 2 == 0 && MI >= 1, "warp tile");
};

__device__ __forceinline__ void named_bar(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }

template <int BM, int BN, int WM, int WN, int KS, int KB, int CK>
__global__ void __launch_bounds__(F64Cfg<BM, BN, WM, WN, KS, KB, CK>::THREADS, 1)
    gemm_f64_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                    const __grid_constant__ CUtensorMap tmA3, const __grid_constant__ CUtensorMap tmB3, GemmArgs args,
                    WorkSched sched) {
  using Cfg = F64Cfg<BM, BN, WM, WN, KS, KB, CK>;
  // optional per-CTA timeline (MM_TRACE=1), globaltimer ns: [0] entry, [1] prologue done, [2] first
  // load issued, [3] first stage landed (consumer warp 0), [4] first item's k-loop done, [5] first
  // item stored, [6] exit
  unsigned long long* tl = args.trace ? args.trace + (size_t)blockIdx.x * 8 : nullptr;
  if (tl && threadIdx.x == 0) tl[0] = globaltimer_ns();
  // clock meter (mm_clock_meter): entry stamps stored at once (no register held over the kernel)
  if (args.clk && threadIdx.x == 0 && blockIdx.x < 4096) {
    args.clk[4 * (size_t)blockIdx.x] = clock64();
    args.clk[4 * (size_t)blockIdx.x + 1] = globaltimer_ns();
  }
  constexpr int NCONS = Cfg::NCONS;
  constexpr int NTILE = Cfg::NTILE;
  constexpr int STAGES = Cfg::STAGES;
  extern __shared__ uint8_t smem_raw[];
  const uint32_t raw_u32 = smem_u32(smem_raw);
  const uint32_t base = (raw_u32 + 1023u) & ~1023u;
  uint8_t* smem = smem_raw + (base - raw_u32);
  const uint32_t sA = base;
  const uint32_t sB = base + STAGES * Cfg::A_BYTES;
  const uint32_t bar0 = smem_u32(smem + STAGES * Cfg::STAGE_BYTES);
  auto full_bar = [&](int s) { return bar0 + 8u * s; };
  auto empty_bar = [&](int s) { return bar0 + 8u * (STAGES + s); };
  volatile unsigned* tick_slot = reinterpret_cast<volatile unsigned*>(smem + STAGES * Cfg::STAGE_BYTES + 1016);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const int c = CK == 1 ? (int)blockIdx.x : (int)blockIdx.x / CK;  // schedule unit: CTA, or cluster (CK > 1)
  const uint32_t krank = CK == 1 ? 0u : __shfl_sync(0xffffffffu, cluster_ctarank(), 0);  // K part of the tile
  const uint32_t xbar = bar0 + 16u * STAGES;  // (CK > 1, rank 0) exchange barrier: rank 1's partial has landed
  // (CK > 1) this CTA's part of a whole tile's k-blocks: halves rounded to whole KB groups
  auto k_part = [&](int& kb0, int& kb1) {
    if constexpr (CK > 1) {
      const int h = ((kb1 - kb0 + 1) / 2 + KB - 1) / KB * KB;
      if (krank == 0) kb1 = min(kb1, kb0 + h);
      else kb0 = min(kb1, kb0 + h);
    }
  };
  const int num_kb = sched.num_kb;
  int* err = args.err;

  if (warp == NCONS && lane == 0) {
    if (KB == 1) {
      tma_prefetch_desc(&tmA);
      tma_prefetch_desc(&tmB);
    } else {
      tma_prefetch_desc(&tmA3);
      tma_prefetch_desc(&tmB3);
    }
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(full_bar(s), 1);
      // KB == 1: one k-block group of warps consumes each slot; KB > 1: every warp arrives once
      // per group of KB slots (on its first slot's barrier)
      mbar_init(empty_bar(s), KB == 1 ? NTILE : NCONS);
    }
    if (CK > 1) mbar_init(xbar, NTILE * 32);  // one arrival per thread of rank 1's tile warps
    fence_mbar_init();
  }
  if constexpr (CK > 1) cluster_sync(); else __syncthreads();
  if (tl && threadIdx.x == 0) tl[1] = globaltimer_ns();

  if (warp == NCONS) {
    // ---------------------------------------------------------------- TMA producer
    if (lane == 0) {
      int stage = 0;
      uint32_t phase = 0;
      bool ok = true;
      int t, kb0, kb1;
      pdl_wait();  // programmatic dependent launch: the prologue above overlapped the previous kernel
      for (int j = 0; ok && sched.item(c, j, t, kb0, kb1); ++j) {
        int tm, tn;
        sched.tile_coords(t, tm, tn);
        k_part(kb0, kb1);
        for (int kb = kb0; kb < kb1; kb += KB) {
          if (!mbar_wait(empty_bar(stage), phase ^ 1u, err, 11)) { ok = false; break; }
          mbar_arrive_expect_tx(full_bar(stage), KB * Cfg::STAGE_BYTES);
          const int k0 = kb * BK;
          if constexpr (KB == 1) {
            tma_load_2d(sA + stage * Cfg::A_BYTES, &tmA, full_bar(stage), k0, tm * BM);
#pragma unroll
            for (int b = 0; b < Cfg::NBBOX; ++b)
              tma_load_2d(sB + stage * Cfg::B_BYTES + b * BBOX_BYTES, &tmB, full_bar(stage), tn * BN + b * 16, k0);
          } else {
            // KB k-slabs of A (k-blocks kb..kb+KB-1) and the KB x 16 rows of all column boxes of B
            tma_load_3d(sA + stage * Cfg::A_BYTES, &tmA3, full_bar(stage), 0, tm * BM, kb);
            tma_load_3d(sB + stage * Cfg::B_BYTES, &tmB3, full_bar(stage), 0, k0, tn * (BN / 16));
          }
          if (tl && j == 0 && kb == kb0) tl[2] = globaltimer_ns();
          stage += KB;
          if (stage == STAGES) { stage = 0; phase ^= 1u; }
        }
      }
      if (tl) tl[7] = globaltimer_ns();  // all loads issued
      pdl_launch_dependents();  // all loads issued: the next launch may start its prologue
    }
  } else {
    // ---------------------------------------------------------------- DMMA consumers
    const int kgrp = (int)warp / NTILE;          // k-block group
    const int wm = ((int)warp % NTILE) / WN;     // rows wm*(BM/WM)
    const int wn = ((int)warp % NTILE) % WN;     // cols wn*(BN/WN)
    double* scr = reinterpret_cast<double*>(smem + STAGES * Cfg::STAGE_BYTES + 1024);
    uint32_t gk = 0;  // running k-block count over this CTA's items (KS groups take gk mod KS)
    const int g = (int)lane >> 2;   // fragment row / column index 0..7
    const int kk = (int)lane & 3;   // fragment k index 0..3
    // Conflict-free fragment loads (LDS.64 is served per half-warp: lanes 0-15 then 16-31).
    // Each DMMA takes the four consecutive k's of its quad; the 8 A rows of a fragment are
    // permuted so a half-warp's rows have (r & 7) ∈ {0,2,4,6} / {1,3,5,7}, and the 8 B
    // columns are permuted to {0,1,8,9,2,3,10,11} (+4 for odd n-tiles) inside a 16-column
    // box; the epilogue writes D back through the same permutations.
    const int arow = (g < 4) ? 2 * g : 2 * (g - 4) + 1;           // A/D row of fragment row g
    const int bcol = (g & 1) + (((g >> 1) & 1) << 3) + ((g >> 2) << 1);  // B column of fragment col g
    const int dcol = ((kk & 1) << 3) + ((kk >> 1) << 1);          // first of this thread's 2 D columns
    // k = qd*4 + kk.  A: row r = wm*BM/2 + mi*8 + arow (r & 7 == arow), 16-B chunk k>>1, half k&1.
    const int a_base0 = (wm * (BM / WM) + arow) * 128 + (kk & 1) * 8;
    const int a_x0 = (kk >> 1) ^ arow;
    // B: column c16 = (ni&1)*4 + bcol in box wn*NI/2 + ni/2; chunk (c16>>1) ^ (k & 7), half c16 & 1.
    const int b_base0 = wn * (Cfg::NI / 2) * Cfg::BOX_STRIDE + kk * 128 + (bcol & 1) * 8;
    const int b_x0 = (bcol >> 1) ^ kk;
    double* C = reinterpret_cast<double*>(args.C);
    double* part = reinterpret_cast<double*>(args.ws);
    const bool vec_ok = ((args.ldc & 1) == 0) && ((reinterpret_cast<uintptr_t>(args.C) & 15) == 0);
    int stage = 0;
    uint32_t phase = 0;
    bool ok = true;
    int t, kb0, kb1;
    for (int j = 0; ok && sched.item(c, j, t, kb0, kb1); ++j) {
      int tm, tn;
      sched.tile_coords(t, tm, tn);
      const bool whole = (kb0 == 0 && kb1 == num_kb);  // (of the tile; CK > 1 splits only whole tiles)
      k_part(kb0, kb1);
      double acc[Cfg::MI][Cfg::NI][2];
#pragma unroll
      for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
        for (int ni = 0; ni < Cfg::NI; ++ni) acc[mi][ni][0] = acc[mi][ni][1] = 0.0;

      // (MM_TRACE: first stage landed — checked here, not in the k-loop, where the trace pointer
      // cost a local-memory reload and a branch per k-block)
      if (tl && warp == 0 && j == 0 && mbar_wait(full_bar(stage), phase, err, 12) && lane == 0) tl[3] = globaltimer_ns();
      for (int kb = kb0; kb < kb1; kb += KB) {
        const int nk = min(KB, kb1 - kb);  // k-blocks in this group (KB == 1: one)
        if (KB == 1 && KS > 1 && (int)(gk % KS) != kgrp) {  // the other warp group's k-block
          ++gk;
          if (++stage == STAGES) { stage = 0; phase ^= 1u; }
          continue;
        }
        if (!mbar_wait(full_bar(stage), phase, err, 12)) { ok = false; break; }
        for (int i = 0; i < nk; ++i) {
        if (KB > 1 && KS > 1 && (int)((gk + i) % KS) != kgrp) continue;  // the other warp group's k-block
        // slot (stage + i): A slab at its own slot; B (KB > 1) at the group's B region, k-block i
        const uint8_t* pa = smem + (stage + i) * Cfg::A_BYTES;
        const uint8_t* pb = smem + STAGES * Cfg::A_BYTES + stage * Cfg::B_BYTES + i * BBOX_BYTES;
        int a_base, a_x, b_base, b_x;
        asm volatile("mov.b32 %0, %1;" : "=r"(a_base) : "r"(a_base0));
        asm volatile("mov.b32 %0, %1;" : "=r"(a_x) : "r"(a_x0));
        asm volatile("mov.b32 %0, %1;" : "=r"(b_base) : "r"(b_base0));
        asm volatile("mov.b32 %0, %1;" : "=r"(b_x) : "r"(b_x0));
#pragma unroll
        for (int qd = 0; qd < 4; ++qd) {
          // Fragment addresses from two thread constants re-materialised per k-block (opaque
          // to the compiler, so it does not hoist 16+ loop-invariant addresses and spill them):
          //   A: pa + a_base + (((qd<<1) ^ a_x) << 4) + mi*1024
          //   B: pb + b_base + (((ni&1)<<1 ^ (qd&1)<<2 ^ b_x) << 4) + (ni>>1)*BBOX + qd*512
          double bf[Cfg::NI];
#pragma unroll
          for (int ni = 0; ni < Cfg::NI; ++ni)
            bf[ni] = *reinterpret_cast<const double*>(
                pb + b_base + ((((ni & 1) << 1) ^ ((qd & 1) << 2) ^ b_x) << 4) + (ni >> 1) * Cfg::BOX_STRIDE + qd * 512);
          const uint8_t* pa_q = pa + a_base + ((((qd << 1) & 7) ^ a_x) << 4) + ((qd << 1) & 8) * 16;
#pragma unroll
          for (int mi = 0; mi < Cfg::MI; ++mi) {
            const double af = *reinterpret_cast<const double*>(pa_q + mi * 1024);  // row + 8*mi keeps r & 7
#pragma unroll
            for (int ni = 0; ni < Cfg::NI; ++ni) dmma_8x8x4(acc[mi][ni][0], acc[mi][ni][1], af, bf[ni]);
          }
        }
        }  // k-blocks of the group
        // The slot is refilled by TMA (async proxy) once all warps arrived: order this warp's
        // shared-memory fragment loads (generic proxy) before that.  Without the proxy fence
        // ptxas issued the arrive while the last A-fragment load was still in flight, and a
        // late warp occasionally read the next k-block's data (wrong rows 56-63 of warp 0).
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(empty_bar(stage));
        gk += nk;
        stage += KB;
        if (stage == STAGES) { stage = 0; phase ^= 1u; }
      }
      if (!ok) break;
      if (tl && warp == 0 && lane == 0 && j == 0) tl[4] = globaltimer_ns();
      if constexpr (KS > 1) {
        // groups 1..KS-1 hand their partial sums to group 0 through shared memory (added in
        // group order: fixed, deterministic)
        if (kgrp >= 1) {
          double* mine = scr + (size_t)(kgrp - 1) * (BM * BN);
#pragma unroll
          for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < Cfg::NI; ++ni) {
              const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
              *reinterpret_cast<double2*>(mine + r * BN + cc) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
            }
        }
        named_bar(2, NCONS * 32);
        if (kgrp == 0) {
          for (int g = 1; g < KS; ++g) {
            const double* other = scr + (size_t)(g - 1) * (BM * BN);
#pragma unroll
            for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
              for (int ni = 0; ni < Cfg::NI; ++ni) {
                const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
                const double2 v = *reinterpret_cast<const double2*>(other + r * BN + cc);
                acc[mi][ni][0] += v.x;
                acc[mi][ni][1] += v.y;
              }
          }
        }
        named_bar(3, NCONS * 32);
        if (kgrp != 0) continue;  // group 0 finishes the tile
      }
      if constexpr (CK > 1) {
        // the tile's K halves: rank 1 stores its partial into rank 0's exchange buffer (distributed
        // shared memory), each thread then arrives (release, cluster scope) on rank 0's barrier;
        // rank 0 waits (acquire) and adds: acc(rank 0's k-blocks) + acc(rank 1's) — fixed order
        const uint32_t xs = smem_u32(smem + STAGES * Cfg::STAGE_BYTES + 1024 + Cfg::SCR_BYTES);
        if (krank != 0) {
          const uint32_t rx = mapa_shared(xs, 0);
#pragma unroll
          for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < Cfg::NI; ++ni) {
              const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
              st_cluster_d2(rx + (uint32_t)(r * BN + cc) * 8u, acc[mi][ni][0], acc[mi][ni][1]);
            }
          mbar_arrive_cluster(mapa_shared(xbar, 0));
          continue;  // rank 0 writes the tile
        }
        if (!mbar_wait_cluster(xbar, 0, args.err, 14)) { ok = false; break; }
#pragma unroll
        for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
          for (int ni = 0; ni < Cfg::NI; ++ni) {
            const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
            const double2 v = *reinterpret_cast<const double2*>(smem + STAGES * Cfg::STAGE_BYTES + 1024 + Cfg::SCR_BYTES +
                                                               (size_t)(r * BN + cc) * 8);
            acc[mi][ni][0] += v.x;
            acc[mi][ni][1] += v.y;
          }
      }

      struct StoreMark {  // first item's results written (any path)
        unsigned long long* tl; bool on;
        __device__ ~StoreMark() { if (on) tl[5] = globaltimer_ns(); }
      } mark{tl, tl != nullptr && warp == 0 && lane == 0 && j == 0};
      if (!whole) {
        // ---- split tile: segments c_first .. c_last of the tail range hold its k-blocks in order
        // (c_first from k-block 0).  Each part takes a ticket; every part but the last to finish
        // publishes its partial tile, and the last one adds them all in segment order (fixed, so
        // run-to-run identical whoever finishes last).  A CTA only waits for parts that took their
        // tickets earlier — running CTAs that are just publishing — never for one that may not have
        // started (the grid need not be co-resident).
        const int64_t ti0 = (int64_t)(t - sched.W * sched.nc) * num_kb;
        const int c_first = sched.tail_cluster_of(ti0);
        const int c_last = sched.tail_cluster_of(ti0 + num_kb - 1);
        const unsigned nparts = (unsigned)(c_last - c_first + 1);
        unsigned* tick = args.flags + t;
        unsigned* pub = args.flags + (size_t)sched.tiles_m * sched.tiles_n + t;
        // two slots per CTA: its first tail segment (role 0) and its last (role 1, holds k-block 0)
        auto slot_of = [&](int cc) { return part + ((size_t)cc * 2 + (cc == c_first ? 1 : 0)) * (BM * BN); };
        if (warp == 0 && lane == 0) *tick_slot = atomic_add_acq_rel_gpu(tick, 1u);
        named_bar(1, NTILE * 32);
        const unsigned tk = *tick_slot;
        named_bar(1, NTILE * 32);
        if (tk + 1u < nparts) {
          // ---- not last: publish the partial tile, then count it
          double* slot = slot_of(c);
#pragma unroll
          for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < Cfg::NI; ++ni) {
              const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
              st_cg_d2(slot + r * BN + cc, make_double2(acc[mi][ni][0], acc[mi][ni][1]));
            }
          __threadfence();
          named_bar(1, NTILE * 32);
          if (warp == 0 && lane == 0) red_release_gpu_add(pub, 1u);
          continue;
        }
        // ---- last: wait for the publications (bounded: their CTAs are running), reset the counters
        if (warp == 0 && lane == 0) {
          if (!counter_wait(pub, nparts - 1u, err, 13)) {
            ok = false;
          } else {
            *(volatile unsigned*)tick = 0u;
            *(volatile unsigned*)pub = 0u;
          }
        }
        // bar.sync is .aligned: warp 0 must reconverge (lane 0 done waiting) before it arrives,
        // else the barrier can release the other warps before the partials are acquired
        __syncwarp();
        named_bar(1, NTILE * 32);
        // acc := part(c_first) + part(c_first+1) + ... + part(c_last).  When this CTA is not c_first,
        // its own part goes through its slot too (each thread re-reads only what it stored itself):
        // the sum then reads every part from the workspace, keeping register pressure at the old level.
        if (c != c_first) {
          double* mine = slot_of(c);
          const double* first = slot_of(c_first);
#pragma unroll
          for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < Cfg::NI; ++ni) {
              const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
              st_cg_d2(mine + r * BN + cc, make_double2(acc[mi][ni][0], acc[mi][ni][1]));
              const double2 v = ld_cg_d2(first + r * BN + cc);
              acc[mi][ni][0] = v.x;
              acc[mi][ni][1] = v.y;
            }
        }
        for (int qq = c_first + 1; qq <= c_last; ++qq) {
          const double* slot = slot_of(qq);
#pragma unroll
          for (int mi = 0; mi < Cfg::MI; ++mi)
#pragma unroll
            for (int ni = 0; ni < Cfg::NI; ++ni) {
              const int r = wm * (BM / WM) + mi * 8 + arow, cc = wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
              const double2 v = ld_cg_d2(slot + r * BN + cc);
              acc[mi][ni][0] += v.x;
              acc[mi][ni][1] += v.y;
            }
        }
      }
      {
        // ---- epilogue: registers -> global (predicated on the ragged edges), β ∈ {0, 1}
#pragma unroll
        for (int mi = 0; mi < Cfg::MI; ++mi) {
          const int64_t row = (int64_t)tm * BM + wm * (BM / WM) + mi * 8 + arow;
          if (row >= args.M) continue;
#pragma unroll
          for (int ni = 0; ni < Cfg::NI; ++ni) {
            const int64_t col = (int64_t)tn * BN + wn * (BN / WN) + (ni >> 1) * 16 + (ni & 1) * 4 + dcol;
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
  }
  __syncwarp();
  // CK > 1: rank 0's exchange buffer is written by rank 1; neither CTA leaves before both are done
  if constexpr (CK > 1) cluster_sync(); else __syncthreads();
  if (tl && threadIdx.x == 0) tl[6] = globaltimer_ns();
  if (args.clk && threadIdx.x == 0 && blockIdx.x < 4096) {
    unsigned long long* r = args.clk + 4 * (size_t)blockIdx.x;
    r[2] = clock64();
    r[3] = globaltimer_ns();
  }
}

template <int BM, int BN, int WM, int WN, int KS, int KB = 1, int CK = 1>
cudaError_t launch_impl(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3, const CUtensorMap& tmB3,
                        const GemmArgs& a, const F64Plan& pl, cudaStream_t s) {
  using Cfg = F64Cfg<BM, BN, WM, WN, KS, KB, CK>;
  auto kern = gemm_f64_kernel<BM, BN, WM, WN, KS, KB, CK>;
  static std::atomic<bool> attr_set[kMaxDevices];  // function attributes are per device
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= kMaxDevices) return cudaErrorInvalidDevice;
  if (!attr_set[dev].load()) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, Cfg::SMEM_BYTES);
    if (e != cudaSuccess) return e;
    attr_set[dev].store(true);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(pl.sched.nc * CK, 1, 1);
  cfg.blockDim = dim3(Cfg::THREADS, 1, 1);
  cfg.dynamicSmemBytes = Cfg::SMEM_BYTES;
  cfg.stream = s;
  cudaLaunchAttribute attr[2];
  int na = 0;
  if (CK > 1) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = CK;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (!knob("MM_NO_PDL")) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, tmA, tmB, tmA3, tmB3, a, pl.sched);
}

}  // namespace

F64Plan f64_plan(int64_t M, int64_t N, int64_t K, int num_sms) {
  F64Plan pl;
  pl.w12 = 0;
  auto tiles = [&](int b) { return ((M + b - 1) / b) * ((N + b - 1) / b); };
  // 128x128 from ~0.6 of a wave of them (16-warp kernels, tools/ab_gpu.py: 96 tiles +2.5 %,
  // 81 even, 64 -5 % vs 64x64); else 32x32 when those fit one wave (every CTA one whole tile,
  // no fix-up: C1 = 64 tiles); else 64x64 (measured: 512^3 20.5 us at 64x64 split vs 26.6 us
  // at 32x32 split).
  pl.bm = pl.bn = 5 * tiles(128) >= 3 * num_sms ? 128 : (tiles(32) <= num_sms ? 32 : 64);
  // 96x128 tiles when they fill the last wave almost exactly and 128x128 ones leave it at most
  // 3/4 full (few waves only: the 24x32 warp tiles are a little less efficient): C2 2000x1500x1750
  // = 294 tiles (1.99 waves) instead of 224 (1.51) -> 335.9 -> 326.7 us (tools/probe83.sh)
  if (pl.bm == 128) {
    const int64_t t96 = ((M + 95) / 96) * ((N + 127) / 128), t128 = tiles(128);
    auto fill = [&](int64_t T) { const int64_t r = T % num_sms; return r == 0 ? 1.0 : (double)r / num_sms; };
    if (t96 <= 4 * (int64_t)num_sms && fill(t96) >= 0.9 && fill(t128) <= 0.75) pl.bm = 96;
  }
  // Round 2: the big-tile kernel is 96x128 with 12 consumer warps of 32x32 (3 per SM sub-partition +
  // the producer: 128 registers instead of the 96 that 17 warps leave, no spill): vs 16 warps on
  // 128x128 / 96x128 tiles, C2 +2.5 %, 4096^3 +0.5 %, 8192^3 +0.2 to +1.3 %, 16384^3 +0.9 %, C5 +0.8 %
  // (profiles/ab_f64_w12_r2t.txt); 128x96 ties at 8192^3+ but loses 12 % on C2, 96x192 with 32x48
  // warp tiles 2-10 % slower (profiles/ab_f64_w12_shapes_r2u.txt).
  if (pl.bm == 128 || pl.bm == 96) {
    pl.bm = 96;
    pl.w12 = 1;
  }
  if (const char* e = knob("MM_F64_TILE")) {  // tuning knob: 32 | 64 | 96 (x128, 16 warps) | 128 | 9612 (default)
    const int v = atoi(e);
    pl.w12 = 0;
    if (v == 32 || v == 64 || v == 128) pl.bm = pl.bn = v;
    if (v == 96) { pl.bm = 96; pl.bn = 128; }
    if (v == 9612) { pl.bm = 96; pl.bn = 128; pl.w12 = 1; }  // (A/B) 12 consumer warps of 32x32
  }
  const int tiles_m = (int)((M + pl.bm - 1) / pl.bm);
  const int tiles_n = (int)((N + pl.bn - 1) / pl.bn);
  const int num_kb = (int)((K + BK - 1) / BK);
  const int64_t T = (int64_t)tiles_m * tiles_n;
  int64_t nc;
  int mode;
  if (T <= num_sms && pl.bm == 32) {
    nc = T;  // one whole tile per CTA
    mode = 0;
  } else {
    // whole-tile waves, then the partial last wave split evenly: each CTA >= 4 k-blocks,
    // each tile at most ~4 contributors
    nc = std::min<int64_t>((int64_t)num_sms, T * 4);
    nc = std::min<int64_t>(nc, std::max<int64_t>(1, T * num_kb / 4));
    mode = 1;
  }
  if (const char* e = knob("MM_F64_STREAMK")) mode = atoi(e) != 0 ? 1 : 0;  // tuning knob
  // small tiles: two k-block groups of warps per CTA (latency-bound DMMA chains)
  pl.ks = pl.bm == 32 ? 2 : 1;
  if (const char* e = knob("MM_F64_KS")) {  // tuning knob: 1 | 2 | 4 (32x32 tiles only)
    const int v = atoi(e);
    pl.ks = (pl.bm == 32 && (v == 2 || v == 4 || v == 8 || v == 44)) ? v : 1;
  }
  // 32x32 whole tiles: 4 k-blocks per TMA load (the caller drops to 1 unless n, p are 16-multiples)
  pl.kb = (pl.bm == 32 && mode == 0 && (pl.ks == 1 || pl.ks == 2)) ? 4 : 1;
  if (const char* e = knob("MM_F64_KB")) pl.kb = (pl.kb == 4 && atoi(e) == 4) ? 4 : 1;  // tuning knob
  // at most half a wave of whole 32x32 tiles: split every tile's K over a 2-CTA cluster (knob MM_F64_CK=1 off)
  pl.ck = (pl.bm == 32 && mode == 0 && 2 * T <= num_sms && pl.ks == 2 && num_kb >= 2) ? 2 : 1;
  if (const char* e = knob("MM_F64_CK")) pl.ck = (pl.ck == 2 && atoi(e) == 2) ? 2 : 1;
  int group_m = 8;
  if (const char* e = knob("MM_F64_GROUP_M")) group_m = atoi(e) > 0 ? atoi(e) : group_m;  // tuning knob
  pl.sched = sched_build(tiles_m, tiles_n, group_m, num_kb, (int)std::max<int64_t>(1, nc), mode);
  // two partial-tile slots per CTA (its first and its last tail segment); tickets + publish counts
  pl.ws_bytes = (size_t)std::max(1, pl.sched.ntc) * 2 * pl.bm * pl.bn * sizeof(double);
  pl.flag_count = (int)(2 * T);
  return pl;
}

void f64_box_dims(const F64Plan& pl, uint32_t* a_box, uint32_t* b_box) {
  a_box[0] = BK;
  a_box[1] = (uint32_t)pl.bm;
  b_box[0] = 16;
  b_box[1] = BK;
}

cudaError_t launch_gemm_f64(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                            const CUtensorMap& tmB3, const GemmArgs& a, const F64Plan& pl, cudaStream_t s) {
  if (pl.bm == 96 && pl.w12) return launch_impl<96, 128, 3, 4, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);
  if (pl.bm == 96) return launch_impl<96, 128, 4, 4, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);
  if (pl.bm == 128) {
    // 16 consumer warps of 32x32 (4 per SM sub-partition, ~96 registers): a warp stalled at a k-block
    // boundary or on a fragment load leaves three others to keep the DMMA pipe busy.  8 warps of
    // 64x32 (MM_F64_W8=1) kept it ~93.6 % busy; 16 warps +2-3 % (C2 344 -> 334 us, 8192^3 31.6 -> 30.9 ms)
    if (knob("MM_F64_W8")) return launch_impl<128, 128, 2, 4, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);  // (A/B knob)
    return launch_impl<128, 128, 4, 4, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);
  }
  if (pl.bm == 64) {  // 16 warps of 16x16 (8 of 32x16 with MM_F64_W8=1): +2-11 % at 512^3-1024^3
    if (knob("MM_F64_W8")) return launch_impl<64, 64, 2, 4, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);  // (A/B knob)
    return launch_impl<64, 64, 4, 4, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);
  }
  if (pl.kb > 1) {  // 32x32, grouped loads (KB = 4 k-blocks per TMA load)
    if (pl.ck == 2 && pl.ks == 2) return launch_impl<32, 32, 2, 2, 2, 4, 2>(tmA, tmB, tmA3, tmB3, a, pl, s);
    if (pl.ks == 2) return launch_impl<32, 32, 2, 2, 2, 4>(tmA, tmB, tmA3, tmB3, a, pl, s);
    return launch_impl<32, 32, 2, 2, 1, 4>(tmA, tmB, tmA3, tmB3, a, pl, s);
  }
  if (pl.ks == 8) return launch_impl<32, 32, 1, 1, 8>(tmA, tmB, tmA3, tmB3, a, pl, s);   // 8 warps, each 32x32 over 1/8 of K
  if (pl.ks == 44) return launch_impl<32, 32, 2, 2, 4>(tmA, tmB, tmA3, tmB3, a, pl, s);  // 16 warps, 16x16 over 1/4 of K
  if (pl.ks == 4) return launch_impl<32, 32, 1, 1, 4>(tmA, tmB, tmA3, tmB3, a, pl, s);   // 4 warps, each 32x32 over 1/4 of K
  if (pl.ck == 2 && pl.ks == 2) return launch_impl<32, 32, 2, 2, 2, 1, 2>(tmA, tmB, tmA3, tmB3, a, pl, s);
  if (pl.ks == 2) return launch_impl<32, 32, 2, 2, 2>(tmA, tmB, tmA3, tmB3, a, pl, s);
  return launch_impl<32, 32, 2, 2, 1>(tmA, tmB, tmA3, tmB3, a, pl, s);
}

}  // namespace mmb
