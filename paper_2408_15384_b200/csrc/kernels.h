// kernels.h — host-side launch interface of the device kernels (internal).
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>
#include <algorithm>
#include <cstdint>

#include "sched.cuh"

namespace mmb {

constexpr int kMaxDevices = 64;  // per-device launch state (function attributes, occupancy)
// device error word value latched by MM_F64_EMU when an operand is Inf or NaN (the pipeline-wait
// timeouts latch small positive codes)
constexpr int kErrNonFinite = 0x4E4F4E46;

// Problem as the kernels see it: C (M×N, leading dim ldc elements) = A (M×K) · B (K×N).
// Paper notation: M = m, K = n, N = p.
struct GemmArgs {
  int64_t M, N, K;
  void* C;
  int64_t ldc;
  int beta_one;  // FP64 only: C += A·B (used by SUMMA panels); 0 = overwrite
  int* err;      // device error word (pipeline timeout codes)
  unsigned* sync;  // [0] wave-barrier arrivals, [1] CTAs done (self-resetting)
  int wave_sync;   // align the k-phase of all tiles once per wave (L2 reuse)
  void* ws;         // FP64 stream-K partial tiles (grid × BM × BN doubles)
  unsigned* flags;  // stream-K per-tile arrival counters (zero between launches)
  int c_tma;        // tcgen05 kernel: C written by TMA stores (C base and pitch 16-B aligned)
  int no_reduce;    // tcgen05 kernel: no TMA reduce-add into C (C in a peer GPU's memory)
  int l2_hint;      // tcgen05 kernel: TMA loads of A evict_last, of B evict_first
  unsigned long long* trace;  // optional per-CTA wait-time counters (16 per CTA), MM_TRACE=1
  int debug;        // diagnostics only (MM_DEBUG): bit 0 = tcgen05 producer skips the operand loads
  int ka;           // tcgen05 kernel: 128-B K atoms per stage (1, or 2 for 256-wide pair tiles)
  int exp;          // schedule experiments that keep results exact (knob MM_EXP, A/B only; 0 = off)
  unsigned long long* clk;  // clock meter (mm_clock_meter): per CTA {clock64, globaltimer} at entry and exit, or null
  // tcgen05 INT8 kernel, MM_F64_EMU's products: store C mod m (bytes in [0, m), C a uint8 matrix)
  // instead of the INT32 values (res_m = 0: INT32 C).  Batched (bat_rows > 0): C and A are stacks
  // of batches of bat_rows rows (a multiple of the tile height), batch b's B starts at row
  // b·bat_krows of the B map, and its modulus is res_mt[b]; else one batch with res_mt[0].
  int res_m;
  int bat_rows, bat_krows;
  int res_mt[16];
  int res_c16t[16];    // 2^16 mod m
  float res_rcpt[16];  // 1 / m
};

// FP64 launch plan (tile shape, stream-K grid, workspace needs).
struct F64Plan {
  int bm, bn;       // CTA tile
  int ks;           // k-block groups of consumer warps (small tiles)
  int kb;           // k-blocks per TMA load (small tiles: 3-D slab maps; 1 = 2-D boxes)
  int ck;           // CTAs per tile along K (2: a cluster splits each tile's K; few small tiles)
  int w12;          // (A/B) 96x128 tiles with 12 consumer warps of 32x32 (128 registers)
  WorkSched sched;  // whole-tile waves + split tail over sched.nc persistent CTAs
  size_t ws_bytes;
  int flag_count;
};
F64Plan f64_plan(int64_t M, int64_t N, int64_t K, int num_sms);

// BF16 (A,B bf16 -> C f32) and INT8 (A,B s8 -> C s32) on tcgen05.
// tmA: dims {K, M} box {128 B of K, 128 rows}; tmB: dims {N, K} box {128 B of N, BK rows}; both SWIZZLE_128B.
// nt: accumulators of N=256 per tile (1: 256-wide tiles, TMEM double-buffered; 2: 512-wide tiles, CG=2 only).
// mc: CTA pairs per cluster sharing B (2: clusters of 4 CTAs, 512-row tiles, B slabs multicast; CG=2 only).
// tmBh: B for N-half tail items (sched.nhalf): int8 — box {64 columns, BK rows}, SWIZZLE_64B; bf16 — tmB.
cudaError_t launch_gemm_tc(bool i8, int cg, int nt, int mc, const CUtensorMap& tmA, const CUtensorMap& tmB,
                           const CUtensorMap& tmC, const CUtensorMap& tmBh, const GemmArgs& a, int num_sms,
                           cudaStream_t s);
// Workspace (stream-K partial slabs) and per-tile counters the launch will use.
void tc_plan_needs(bool i8, int cg, int nt, int mc, int ka, int64_t M, int64_t N, int64_t K, int num_sms,
                   size_t* ws_bytes, size_t* flag_count);
// Box extents the tensor maps must be encoded with.
void tc_box_dims(bool i8, int cg, int mc, int ka, uint32_t* a_box /*[2]*/, uint32_t* b_box /*[2]*/);
// Co-resident clusters of the given configuration (0 if the query failed).
int max_clusters(bool i8, int cg, int nt, int mc, int ka, int num_sms);

// FP64 on DMMA (mma.sync m8n8k4) with TMA-fed smem ring.
// tmA3 / tmB3: the 3-D slab maps used when pl.kb > 1 (A {16, m, n/16} box {16, bm, kb};
// B {16, n, p/16} box {16, 16 kb, bn/16}); pass tmA / tmB otherwise.
cudaError_t launch_gemm_f64(const CUtensorMap& tmA, const CUtensorMap& tmB, const CUtensorMap& tmA3,
                            const CUtensorMap& tmB3, const GemmArgs& a, const F64Plan& pl, cudaStream_t s);
void f64_box_dims(const F64Plan& pl, uint32_t* a_box, uint32_t* b_box);

// Copy a rows×cols matrix (pitch src_ld elements) into dst (pitch dst_ld >= cols), zero-filling
// columns [cols, dst_ld).  esize ∈ {1, 2, 8}.  Coalesced 16-byte stores on the destination.
cudaError_t launch_pack_pad(const void* src, int64_t rows, int64_t cols, int64_t src_ld, void* dst, int64_t dst_ld,
                            int esize, cudaStream_t s);

}  // namespace mmb
