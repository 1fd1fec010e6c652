// mm_abi.cu — the C-ABI (include/mm.h): argument validation, context, the
// planner that picks a kernel and encodes TMA tensor maps, the padding edge
// path, and the host-buffer pipeline.
//
// Operation: C = A·B, A m×n, B n×p, row-major.
#include <dlfcn.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <vector>

#include "ctx.h"
#include "kernels.h"
#include "knobs.h"

#define MM_VERSION "0.1.0"

namespace mmb {

mm_status set_err(mm_ctx* ctx, mm_status s, const char* fmt, ...) {
  if (ctx) {
    char buf[768];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    ctx->last_error = buf;
  }
  return s;
}

size_t dtype_in_size(mm_dtype t) { return (t == MM_F64 || t == MM_F64_EMU) ? 8 : (t == MM_BF16_F32 ? 2 : 1); }
size_t dtype_out_size(mm_dtype t) { return (t == MM_F64 || t == MM_F64_EMU) ? 8 : 4; }

mm_status ensure_buffer(mm_ctx* ctx, void** buf, size_t* have, size_t need) {
  if (*have >= need && *buf) return MM_OK;
  if (*buf) {
    cudaDeviceSynchronize();
    cudaFree(*buf);
    *buf = nullptr;
    *have = 0;
  }
  size_t sz = need < 256 ? 256 : need;
  if (cudaMalloc(buf, sz) != cudaSuccess) {
    cudaGetLastError();
    *buf = nullptr;
    return set_err(ctx, MM_ERR_WORKSPACE, "cudaMalloc(%zu bytes) failed", sz);
  }
  *have = sz;
  return MM_OK;
}

namespace {

// ---- cuTensorMapEncodeTiled, resolved at run time from the driver (no link-time libcuda).
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
EncodeTiledFn g_encode = nullptr;
std::once_flag g_encode_once;

EncodeTiledFn get_encode() {
  std::call_once(g_encode_once, [] {
    void* fn = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &fn, 12000, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      g_encode = reinterpret_cast<EncodeTiledFn>(fn);
    else
      cudaGetLastError();
  });
  return g_encode;
}

// Tensor-map cache lookup / insert (ctx->map_cache).
bool map_cache_get(mm_ctx* ctx, const uint64_t (&key)[8], CUtensorMap* out) {
  for (int i = 0; i < ctx->map_cache_used; ++i)
    if (memcmp(ctx->map_cache[i].key, key, sizeof key) == 0) {
      *out = ctx->map_cache[i].map;
      return true;
    }
  return false;
}
void map_cache_put(mm_ctx* ctx, const uint64_t (&key)[8], const CUtensorMap& m) {
  const int n = sizeof(ctx->map_cache) / sizeof(ctx->map_cache[0]);
  const int i = ctx->map_cache_used < n ? ctx->map_cache_used++ : (ctx->map_cache_next++ % n);
  memcpy(ctx->map_cache[i].key, key, sizeof key);
  ctx->map_cache[i].map = m;
}

// Row-major rows×cols matrix with pitch `ld` elements → 2-D tensor map {cols, rows}.
mm_status encode_2d(mm_ctx* ctx, CUtensorMap* map, CUtensorMapDataType dt, size_t esz, const void* ptr, int64_t rows,
                    int64_t cols, int64_t ld, const uint32_t box[2], const char* what, int swizzle_bytes = 128) {
  const uint64_t key[8] = {2, (uint64_t)(uintptr_t)ptr, (uint64_t)rows, (uint64_t)cols, (uint64_t)ld,
                           ((uint64_t)box[0] << 32) | box[1], ((uint64_t)dt << 32) | (uint64_t)esz, (uint64_t)swizzle_bytes};
  if (map_cache_get(ctx, key, map)) return MM_OK;
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_err(ctx, MM_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)(ld * (int64_t)esz)};
  cuuint32_t boxd[2] = {box[0], box[1]};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = enc(map, dt, 2, const_cast<void*>(ptr), dims, strides, boxd, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   swizzle_bytes == 0    ? CU_TENSOR_MAP_SWIZZLE_NONE
                   : swizzle_bytes == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                         : CU_TENSOR_MAP_SWIZZLE_128B,
                   CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(ctx, MM_ERR_UNSUPPORTED, "TMA encode failed for %s (%lld x %lld, ld %lld): CUresult %d", what,
                   (long long)rows, (long long)cols, (long long)ld, (int)r);
  map_cache_put(ctx, key, *map);
  return MM_OK;
}

// Row-major rows x cols matrix (pitch ld elements) seen as 3-D {16, rows, cols/16}: element
// (r, 16*o + i) at dims (i, r, o) — one box covers several consecutive 16-column slabs (cols % 16 == 0).
mm_status encode_3d_slabs(mm_ctx* ctx, CUtensorMap* map, const void* ptr, int64_t rows, int64_t cols, int64_t ld,
                          const uint32_t box[3], const char* what) {
  const uint64_t key[8] = {3, (uint64_t)(uintptr_t)ptr, (uint64_t)rows, (uint64_t)cols, (uint64_t)ld,
                           ((uint64_t)box[0] << 32) | box[1], (uint64_t)box[2], 0};
  if (map_cache_get(ctx, key, map)) return MM_OK;
  EncodeTiledFn enc = get_encode();
  if (!enc) return set_err(ctx, MM_ERR_RUNTIME, "cuTensorMapEncodeTiled unavailable from the driver");
  cuuint64_t dims[3] = {16, (cuuint64_t)rows, (cuuint64_t)(cols / 16)};
  cuuint64_t strides[2] = {(cuuint64_t)(ld * 8), 128};
  cuuint32_t boxd[3] = {box[0], box[1], box[2]};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, const_cast<void*>(ptr), dims, strides, boxd, estr,
                   CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                   CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS)
    return set_err(ctx, MM_ERR_UNSUPPORTED, "TMA 3-D encode failed for %s (%lld x %lld, ld %lld): CUresult %d", what,
                   (long long)rows, (long long)cols, (long long)ld, (int)r);
  map_cache_put(ctx, key, *map);
  return MM_OK;
}

inline bool tma_ok(const void* p, int64_t ld, size_t esz) {
  return (reinterpret_cast<uintptr_t>(p) % 16 == 0) && ((ld * (int64_t)esz) % 16 == 0);
}
inline int64_t round_up(int64_t x, int64_t a) { return (x + a - 1) / a * a; }

bool ranges_overlap(const void* a, size_t abytes, const void* b, size_t bbytes) {
  const uintptr_t a0 = reinterpret_cast<uintptr_t>(a), b0 = reinterpret_cast<uintptr_t>(b);
  return a0 < b0 + bbytes && b0 < a0 + abytes;
}

int force_cg() {
  const char* e = knob("MM_FORCE_CG");
  if (!e) return 0;
  int v = atoi(e);
  return (v == 1 || v == 2) ? v : 0;
}

}  // namespace

// Diagnostic knobs (MM_DEBUG skips operand loads or output stores — results are garbage by design;
// MM_TRACE / MM_HOST_TRACE synchronize the stream to print timelines) exist only in the diagnostic
// build (`make diag` -> libmm_b200_diag.so, -DMM_DIAG).  The release library refuses them.
mm_status refuse_diag_knobs(mm_ctx* ctx) {
#ifndef MM_DIAG
  for (const char* k : {"MM_DEBUG", "MM_TRACE", "MM_HOST_TRACE"})
    if (knob(k))
      return set_err(ctx, MM_ERR_UNSUPPORTED, "%s is a diagnostic knob of the diagnostic build only (make diag, "
                     "MM_B200_LIB=.../libmm_b200_diag.so); unset it for the release library", k);
#else
  (void)ctx;
#endif
  return MM_OK;
}

namespace {
// The context's scratch (wave-barrier counters, split-tile tickets and slabs, padding buffer) is
// shared by its launches, so they must not overlap: a product enqueued on a stream other than the
// previous product's waits for that one first (one event per context).  Inside a CUDA-graph capture
// the caller owns the ordering (no cross-capture events).
bool capturing(cudaStream_t s) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cs) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return cs != cudaStreamCaptureStatusNone;
}
mm_status order_after_previous(mm_ctx* ctx, cudaStream_t s, bool cap) {
  if (cap || !ctx->ev_last_valid || s == ctx->last_stream) return MM_OK;
  if (cudaStreamWaitEvent(s, ctx->ev_last, 0) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "cross-stream ordering failed: %s", cudaGetErrorString(cudaGetLastError()));
  return MM_OK;
}
mm_status record_launch(mm_ctx* ctx, cudaStream_t s, bool cap) {
  if (cap) return MM_OK;
  if (!ctx->ev_last && cudaEventCreateWithFlags(&ctx->ev_last, cudaEventDisableTiming) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "event creation failed");
  if (cudaEventRecord(ctx->ev_last, s) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "event record failed: %s", cudaGetErrorString(cudaGetLastError()));
  ctx->last_stream = s;
  ctx->ev_last_valid = true;
  return MM_OK;
}
}  // namespace

mm_status gemm_ld_impl(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, const void* A, int64_t lda,
                       const void* B, int64_t ldb, void* C, int64_t ldc, int beta_one, cudaStream_t s);

mm_status gemm_ld(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, int beta_one, cudaStream_t s) {
  const bool cap = capturing(s);
  mm_status st = order_after_previous(ctx, s, cap);
  if (st != MM_OK) return st;
  st = gemm_ld_impl(ctx, m, n, p, dtype, A, lda, B, ldb, C, ldc, beta_one, s);
  if (st != MM_OK) return st;
  return record_launch(ctx, s, cap);
}

mm_status gemm_ld_impl(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, const void* A, int64_t lda,
                       const void* B, int64_t ldb, void* C, int64_t ldc, int beta_one, cudaStream_t s) {
  if (dtype == MM_F64_EMU)
    return gemm_f64_emu(ctx, m, n, p, static_cast<const double*>(A), lda, static_cast<const double*>(B), ldb,
                        static_cast<double*>(C), ldc, beta_one, s);
  const size_t esz = dtype_in_size(dtype);
  // persistent grids over the SMs not reserved for concurrent (communication) kernels
  const int num_sms = std::max(4, (ctx->num_sms - std::max(0, ctx->sm_reserve)) & ~1);
  // ---- edge path: operands TMA cannot read in place are copied to a zero-padded pitch.
  const bool padA = !tma_ok(A, lda, esz);
  const bool padB = !tma_ok(B, ldb, esz);
  const int64_t align_el = 16 / (int64_t)esz;
  const int64_t ldA2 = padA ? round_up(n, align_el) : lda;
  const int64_t ldB2 = padB ? round_up(p, align_el) : ldb;
  const size_t bytesA = padA ? (size_t)round_up((int64_t)(m * ldA2 * esz), 256) : 0;
  const size_t bytesB = padB ? (size_t)round_up((int64_t)(n * ldB2 * esz), 256) : 0;
  const void* Ause = A;
  const void* Buse = B;
  if (padA || padB) {
    const size_t need = bytesA + bytesB;
    uint8_t* ws;
    if (ctx->user_ws && ctx->user_ws_bytes >= need && (reinterpret_cast<uintptr_t>(ctx->user_ws) % 256) == 0) {
      ws = static_cast<uint8_t*>(ctx->user_ws);
    } else {
      mm_status st = ensure_buffer(ctx, &ctx->ws, &ctx->ws_bytes, need);
      if (st != MM_OK) return st;
      ws = static_cast<uint8_t*>(ctx->ws);
    }
    if (padA) {
      if (launch_pack_pad(A, m, n, lda, ws, ldA2, (int)esz, s) != cudaSuccess)
        return set_err(ctx, MM_ERR_RUNTIME, "pack(A) launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      ++ctx->launches;
      Ause = ws;
    }
    if (padB) {
      if (launch_pack_pad(B, n, p, ldb, ws + bytesA, ldB2, (int)esz, s) != cudaSuccess)
        return set_err(ctx, MM_ERR_RUNTIME, "pack(B) launch failed: %s", cudaGetErrorString(cudaGetLastError()));
      ++ctx->launches;
      Buse = ws + bytesA;
    }
  }

  GemmArgs a;
  a.M = m;
  a.N = p;
  a.K = n;
  a.C = C;
  a.ldc = ldc;
  a.beta_one = beta_one;
  a.err = ctx->d_err;
  a.sync = reinterpret_cast<unsigned*>(ctx->d_err + 1);
  // The k-phase barrier pays off only when the operands do not fit in L2 (126 MB):
  // then the tiles of a wave must walk K together to share A/B slabs.
  const double operand_bytes = (double)(m * n + n * p) * (double)esz;
  int wave_sync = ctx->wave_sync;
  if (const char* e = knob("MM_WAVE_SYNC")) wave_sync = atoi(e);  // tuning knob (0 off, 1 auto, 2 on)
  a.wave_sync = wave_sync == 1 ? (operand_bytes > 96.0 * (1 << 20)) : (wave_sync > 1);

  CUtensorMap tmA, tmB;
  uint32_t abox[2], bbox[2];
  cudaError_t e;
  a.ws = nullptr;
  a.flags = nullptr;
  a.c_tma = 0;
  // C in another process's (a peer GPU's) memory: plain stores only, no TMA reduce-add split tail
  a.no_reduce = ctx->c_remote;
  for (const auto& mp : ctx->ipc_open)
    if (reinterpret_cast<const uint8_t*>(C) >= static_cast<const uint8_t*>(mp.base) &&
        reinterpret_cast<const uint8_t*>(C) < static_cast<const uint8_t*>(mp.base) + std::max<size_t>(mp.bytes, 1))
      a.no_reduce = 1;
  // L2 eviction hints on the operand loads: measured no gain (A evict_last) or a loss
  // (B evict_first: C4 DRAM reads 8.9 -> 12.7 GB), so off unless requested.
  a.l2_hint = 0;
  a.trace = nullptr;
  a.debug = 0;
  a.ka = 1;
  a.clk = ctx->clk_on ? ctx->clk_buf : nullptr;
  a.res_m = 0;
  a.bat_rows = 0;
  a.bat_krows = 0;
#ifdef MM_DIAG
  if (const char* env = knob("MM_DEBUG")) a.debug = atoi(env);  // diagnostics: results are garbage
  const bool trace = knob("MM_TRACE") != nullptr && dtype != MM_F64;  // debug: per-role wait times
#else
  const bool trace = false;
#endif
  int trace_nt = 0, trace_mc = 0, trace_maxcl = 0;
  if (trace) {
    if (!ctx->trace_buf && cudaMalloc(&ctx->trace_buf, 4096 * 48 * sizeof(unsigned long long)) != cudaSuccess)
      return set_err(ctx, MM_ERR_WORKSPACE, "trace buffer allocation failed");
    cudaMemsetAsync(ctx->trace_buf, 0, 4096 * 48 * sizeof(unsigned long long), s);
    a.trace = static_cast<unsigned long long*>(ctx->trace_buf);
  }
  if (const char* env = knob("MM_L2_HINT")) a.l2_hint = atoi(env);  // tuning knob
  a.exp = 0;
  if (const char* env = knob("MM_EXP")) a.exp = atoi(env);  // (A/B knob: schedule experiments)
  // stream-K workspace (partial tiles) + self-resetting per-tile counters, shared by both kernels
  auto ensure_sk = [&](size_t ws_bytes, size_t flag_count) -> mm_status {
    if (ctx->sk_flag_count < flag_count) {
      if (ctx->sk_flags) {
        cudaDeviceSynchronize();
        cudaFree(ctx->sk_flags);
        ctx->sk_flags = nullptr;
        ctx->sk_flag_count = 0;
      }
      if (cudaMalloc(&ctx->sk_flags, flag_count * sizeof(unsigned)) != cudaSuccess ||
          cudaMemset(ctx->sk_flags, 0, flag_count * sizeof(unsigned)) != cudaSuccess)
        return set_err(ctx, MM_ERR_WORKSPACE, "stream-K counter allocation failed");
      ctx->sk_flag_count = flag_count;
    }
    if (ws_bytes) {
      mm_status wst = ensure_buffer(ctx, &ctx->sk_ws, &ctx->sk_ws_bytes, ws_bytes);
      if (wst != MM_OK) return wst;
    }
    a.ws = ctx->sk_ws;
    a.flags = ctx->sk_flags;
    return MM_OK;
  };
  if (dtype == MM_F64) {
    F64Plan pl = f64_plan(m, p, n, num_sms);
    if (pl.kb > 1 && (n % 16 != 0 || p % 16 != 0)) pl.kb = 1;  // grouped loads need exact 16-slabs
    mm_status st = ensure_sk(pl.ws_bytes, (size_t)pl.flag_count);
    if (st != MM_OK) return st;
    f64_box_dims(pl, abox, bbox);
    st = encode_2d(ctx, &tmA, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Ause, m, n, padA ? ldA2 : lda, abox, "A");
    if (st != MM_OK) return st;
    st = encode_2d(ctx, &tmB, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 8, Buse, n, p, padB ? ldB2 : ldb, bbox, "B");
    if (st != MM_OK) return st;
#ifdef MM_DIAG
    const bool ftrace = knob("MM_TRACE") != nullptr;
#else
    const bool ftrace = false;
#endif
    if (ftrace) {
      if (!ctx->trace_buf && cudaMalloc(&ctx->trace_buf, 4096 * 48 * sizeof(unsigned long long)) != cudaSuccess)
        return set_err(ctx, MM_ERR_WORKSPACE, "trace buffer allocation failed");
      cudaMemsetAsync(ctx->trace_buf, 0, 4096 * 8 * sizeof(unsigned long long), s);
      a.trace = static_cast<unsigned long long*>(ctx->trace_buf);
    }
    // small tiles: several k-blocks per TMA load (3-D slab maps), when K and p are 16-multiples
    CUtensorMap tmA3 = tmA, tmB3 = tmB;
    if (pl.kb > 1) {
      const uint32_t a3[3] = {16, (uint32_t)pl.bm, (uint32_t)pl.kb};
      const uint32_t b3[3] = {16, (uint32_t)(16 * pl.kb), (uint32_t)(pl.bn / 16)};
      st = encode_3d_slabs(ctx, &tmA3, Ause, m, n, padA ? ldA2 : lda, a3, "A (k-slab groups)");
      if (st != MM_OK) return st;
      st = encode_3d_slabs(ctx, &tmB3, Buse, n, p, padB ? ldB2 : ldb, b3, "B (column-slab groups)");
      if (st != MM_OK) return st;
    }
    e = launch_gemm_f64(tmA, tmB, tmA3, tmB3, a, pl, s);
    if (e == cudaSuccess && ftrace) {
      std::vector<unsigned long long> h(4096 * 8);
      cudaStreamSynchronize(s);
      cudaMemcpy(h.data(), ctx->trace_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
      unsigned long long e0 = ~0ull;
      for (int c = 0; c < pl.sched.nc; ++c) if (h[(size_t)c * 8]) e0 = std::min(e0, h[(size_t)c * 8]);
      double acc[8] = {0};
      int cnt[8] = {0};
      for (int c = 0; c < pl.sched.nc; ++c)
        for (int k = 0; k < 8; ++k)
          if (h[(size_t)c * 8 + k]) { acc[k] += (double)(h[(size_t)c * 8 + k] - e0); ++cnt[k]; }
      fprintf(stderr, "[mm trace f64] m=%lld n=%lld p=%lld tile %d ks %d CTAs %d | us after first entry (CTA avg): entry %.2f "
              "prologue %.2f first-load %.2f first-data %.2f k-loop-done %.2f stored %.2f exit %.2f | loads issued %.2f\n",
              (long long)m, (long long)n, (long long)p, pl.bm, pl.ks, pl.sched.nc,
              cnt[0] ? 1e-3 * acc[0] / cnt[0] : 0.0, cnt[1] ? 1e-3 * acc[1] / cnt[1] : 0.0,
              cnt[2] ? 1e-3 * acc[2] / cnt[2] : 0.0, cnt[3] ? 1e-3 * acc[3] / cnt[3] : 0.0,
              cnt[4] ? 1e-3 * acc[4] / cnt[4] : 0.0, cnt[5] ? 1e-3 * acc[5] / cnt[5] : 0.0,
              cnt[6] ? 1e-3 * acc[6] / cnt[6] : 0.0, cnt[7] ? 1e-3 * acc[7] / cnt[7] : 0.0);
    }
  } else {
    if (beta_one) return set_err(ctx, MM_ERR_UNSUPPORTED, "accumulate (beta=1) is only implemented for MM_F64");
    const bool i8 = dtype == MM_S8_S32;
    int cg = force_cg();
    if (!cg) cg = (m <= 128) ? 1 : 2;
    if (ctx->res_mod && ctx->res_nbat > 1) cg = 2;  // batched residue products: 256-row pair tiles
    // 512-wide tiles (two N=256 accumulators per CTA pair) for large operands: 25 % fewer
    // L2->SM bytes and DRAM re-reads per FLOP, at the price of no TMEM double-buffering.
    // ... and whenever they fill at least one wave of the pairs (measured 4096^3: int8 +3 %,
    // bf16 +6 %; 2048^3, 32 wide tiles for 74 pairs: -25 %, tools/ab_gpu.py).  Even with a
    // ragged last wave they win at burst clocks: the 8-GPU row block of C4 (2048 x 16384 x
    // 16384, 3.46 waves of 512-wide tiles vs 6.92 of 256-wide ones) runs 6 % faster at NT=2.
    const int64_t tiles_nt2 = ((m + 255) / 256) * ((p + 511) / 512);
    int nt = (cg == 2 && (a.wave_sync || tiles_nt2 >= num_sms / 2)) ? 2 : 1;
    // two CTA pairs per cluster sharing (multicasting) every B slab
    int mc = 1;
    if (const char* env = knob("MM_MC")) mc = (cg == 2 && m > 256 && atoi(env) == 2) ? 2 : 1;  // tuning knob
    if (ctx->res_mod && ctx->res_nbat > 1) mc = 1;  // batched residue products: one pair per tile
    // With few waves of 512-wide tiles (quantisation, an exposed read-out per tile) 256-wide tiles
    // with TMEM double-buffering and two K atoms per stage win: int8 4096^3 +3 %, bf16 4096^3 +2 %;
    // from ~7 waves on (8192^3) 512-wide tiles stay ahead (tools/ab_gpu.py).
    // Round 2 (after the warp-elected MMA issue, 256- and 512-wide tiles run at the same rate per
    // FLOP up to ~8 waves): pick the width with fewer rounds of work per cluster; 256-wide rounds
    // count half, a partial last round of them that fits the N-half split (tail <= nc/2) 0.4;
    // ties go to 512-wide tiles (fewer DRAM re-reads).  Measured: int8 4096x4096x8192 / 8192x4096x4096
    // +14 / +16 %, bf16 4096x4096x8192 +4 % (3.46 waves of 512-wide tiles: 4 rounds vs 3.5);
    // int8 6144^3 equal (4 vs 4) (profiles/ab_nt_rounds_r2zi.txt).
    if (nt == 2 && !a.wave_sync && mc == 1) {
      const int64_t nc = std::max(1, num_sms / 2);
      const int64_t tiles_nt1 = ((m + 255) / 256) * ((p + 255) / 256);
      const double r2 = (double)((tiles_nt2 + nc - 1) / nc);
      const int64_t tail1 = tiles_nt1 % nc;
      const double r1 = 0.5 * (double)(tiles_nt1 / nc) + (tail1 == 0 ? 0.0 : (2 * tail1 <= nc ? 0.4 : 0.5));
      if (r1 < r2) nt = 1;
    }
    if (const char* env = knob("MM_NT")) nt = (cg == 2 && atoi(env) == 2) ? 2 : 1;  // tuning knob
    // 256-wide pair tiles: two 128-B K atoms per stage — 8 MMAs per barrier wait and commit instead
    // of 4 (the single issuing thread, not the tensor pipe, bounded 4-MMA stages at ~75 % busy)
    a.ka = (cg == 2 && nt == 1 && n >= 8 * (i8 ? 128 : 64)) ? 2 : 1;
    if (const char* env = knob("MM_KA")) a.ka = (cg == 2 && nt == 1 && atoi(env) == 2) ? 2 : 1;
    size_t ws_bytes = 0, flag_count = 0;
    tc_plan_needs(i8, cg, nt, mc, a.ka, m, p, n, num_sms, &ws_bytes, &flag_count);
    mm_status st = ensure_sk(ws_bytes, flag_count);
    if (st != MM_OK) return st;
    tc_box_dims(i8, cg, mc, a.ka, abox, bbox);
    const CUtensorMapDataType dt = i8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    st = encode_2d(ctx, &tmA, dt, esz, Ause, m, n, padA ? ldA2 : lda, abox, "A");
    if (st != MM_OK) return st;
    // batched residue products (MM_F64_EMU): B is a stack of res_nbat batches of res_bat_krows rows
    const int64_t brows = ctx->res_mod && ctx->res_nbat > 1 ? (int64_t)ctx->res_nbat * ctx->res_bat_krows : n;
    st = encode_2d(ctx, &tmB, dt, esz, Buse, brows, p, padB ? ldB2 : ldb, bbox, "B");
    if (st != MM_OK) return st;
    // C through TMA stores when its base and pitch allow (else predicated register stores)
    CUtensorMap tmC;
    memset(&tmC, 0, sizeof tmC);
    if (ctx->res_mod) {  // MM_F64_EMU's products: C mod res_mod as bytes (uint8 C, TMA stores only)
      if (!i8 || !tma_ok(C, ldc, 1))
        return set_err(ctx, MM_ERR_RUNTIME, "internal: residue output needs an INT8 product and a TMA-storable C");
      a.res_m = 1;
      const int nb = ctx->res_nbat > 1 ? ctx->res_nbat : 1;
      for (int b = 0; b < 16; ++b) {
        const int md = b < nb ? (nb > 1 ? ctx->res_mods[b] : ctx->res_mod) : 1;
        a.res_mt[b] = md;
        a.res_c16t[b] = (int)(65536u % (unsigned)md);
        a.res_rcpt[b] = 1.0f / (float)md;
      }
      if (nb > 1) {  // batches stacked along M: whole 256-row pair tiles per batch, no multicast clusters
        if (ctx->res_bat_rows % 256 != 0 || cg != 2 || mc != 1 || padB)
          return set_err(ctx, MM_ERR_RUNTIME, "internal: batched residue products need 256-row batches and CTA pairs");
        a.bat_rows = (int)ctx->res_bat_rows;
        a.bat_krows = (int)ctx->res_bat_krows;
      }
      a.no_reduce = 1;  // partial sums are added before the reduction, never in C
      a.c_tma = 1;
      const uint32_t rbox[2] = {32, 32};
      st = encode_2d(ctx, &tmC, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, C, m, p, ldc, rbox, "C residues", 0);
      if (st != MM_OK) return st;
    } else {
    a.c_tma = tma_ok(C, ldc, 4) ? 1 : 0;
    if (const char* env = knob("MM_TMA_STORE")) a.c_tma = a.c_tma && atoi(env) != 0;  // tuning knob
    if (a.c_tma) {
      const uint32_t cbox[2] = {32, 32};
      st = encode_2d(ctx, &tmC, i8 ? CU_TENSOR_MAP_DATA_TYPE_INT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, C, m, p, ldc,
                     cbox, "C");
      if (st != MM_OK) return st;
    }
    }
    // B for N-half tail items: bf16 — the same map (a 64-column box is 128 B); int8 — 64-column
    // (64-B) boxes, 64-byte swizzle
    CUtensorMap tmBh = tmB;
    if (i8 && cg == 2 && nt == 1 && mc == 1) {
      const uint32_t hbox[2] = {64, bbox[1]};
      st = encode_2d(ctx, &tmBh, dt, esz, Buse, brows, p, padB ? ldB2 : ldb, hbox, "B (64-column boxes)", 64);
      if (st != MM_OK) return st;
    }
    e = launch_gemm_tc(i8, cg, nt, mc, tmA, tmB, tmC, tmBh, a, num_sms, s);
    trace_nt = nt;
    trace_mc = mc;
    if (trace) trace_maxcl = max_clusters(i8, cg, nt, mc, a.ka, num_sms);
  }
  if (e == cudaSuccess) ++ctx->launches;
  if (e == cudaSuccess && trace) {
    // CTA-average wait times by role, as fractions of the kernel's span (stderr)
    std::vector<unsigned long long> h(4096 * 48);
    cudaStreamSynchronize(s);
    cudaMemcpy(h.data(), ctx->trace_buf, h.size() * sizeof(unsigned long long), cudaMemcpyDeviceToHost);
    unsigned long long t0 = ~0ull, t1 = 0;
    double sum[6] = {0, 0, 0, 0, 0, 0}, chunk[5] = {0, 0, 0, 0, 0}, clk_cyc = 0, clk_ns = 0;
    int nct = 0, nmma = 0;
    for (int c = 0; c < 4096; ++c) {
      const unsigned long long* r = &h[(size_t)c * 16];
      if (r[6]) {
        t0 = std::min(t0, r[6]);
        t1 = std::max(t1, r[7]);
        ++nmma;
        if (r[7] > r[6]) { clk_cyc += (double)r[13]; clk_ns += (double)(r[7] - r[6]); }
      }
      if (r[0] || r[1] || r[4]) ++nct;
      for (int k = 0; k < 6; ++k) sum[k] += (double)r[k];
      for (int k = 0; k < 5; ++k) chunk[k] += (double)r[8 + k];
    }
    {
      // average timeline of the MMA-issuing CTAs, relative to the earliest kernel entry (us)
      unsigned long long e0 = ~0ull;
      for (int c = 0; c < 4096; ++c)
        if (h[(size_t)c * 16 + 14]) e0 = std::min(e0, h[(size_t)c * 16 + 14]);
      double acc[32] = {0};
      int cnt[32] = {0};
      double ent = 0, setup = 0, pdl = 0, ex = 0, exmax = 0;
      int nent = 0;
      for (int c = 0; c < 4096; ++c) {
        const unsigned long long* r = &h[(size_t)c * 16];
        const unsigned long long* tlc = &h[4096 * 16 + (size_t)c * 32];
        if (!r[6]) continue;
        ent += (double)(r[14] - e0);
        setup += (double)(r[6] - e0);
        if (r[15]) pdl += (double)(r[15] - e0);
        ex += (double)(r[7] - e0);
        exmax = std::max(exmax, (double)(r[7] - e0));
        ++nent;
        for (int k = 0; k < 32; ++k)
          if (tlc[k]) { acc[k] += (double)(tlc[k] - e0); ++cnt[k]; }
      }
      if (nent) {
        fprintf(stderr, "[mm trace] timeline (us after first CTA entry, CTA average): entry %.2f setup %.2f pdl-wait %.2f "
                "exit %.2f (last %.2f)", 1e-3 * ent / nent, 1e-3 * setup / nent, 1e-3 * pdl / nent, 1e-3 * ex / nent,
                1e-3 * exmax);
        for (int j = 0; j < 8; ++j)
          if (cnt[4 * j])
            fprintf(stderr, " | item %d: MMA %.2f-%.2f epi %.2f-%.2f (%d)", j, 1e-3 * acc[4 * j] / cnt[4 * j],
                    cnt[4 * j + 1] ? 1e-3 * acc[4 * j + 1] / cnt[4 * j + 1] : 0.0,
                    cnt[4 * j + 2] ? 1e-3 * acc[4 * j + 2] / cnt[4 * j + 2] : 0.0,
                    cnt[4 * j + 3] ? 1e-3 * acc[4 * j + 3] / cnt[4 * j + 3] : 0.0, cnt[4 * j]);
        fprintf(stderr, "\n");
      }
    }
    if (clk_ns > 0) fprintf(stderr, "[mm trace] effective SM clock during the kernel %.0f MHz\n", 1e3 * clk_cyc / clk_ns);
    if (chunk[4] > 0)
      fprintf(stderr, "[mm trace] epilogue cycles per 4-KB chunk (warp 2): tmem-ld wait %.0f, st.shared %.0f, "
              "proxy fence %.0f, store issue %.0f\n", chunk[0] / chunk[4], chunk[1] / chunk[4], chunk[2] / chunk[4],
              chunk[3] / chunk[4]);
    const double span = (double)(t1 - t0);
    if (nct && nmma && span > 0)
      fprintf(stderr,
              "[mm trace] m=%lld n=%lld p=%lld nt=%d mc=%d mma-issuing CTAs %d (max resident clusters %d) span %.1f us | producer: wave-barrier %.2f%% empty-slot %.2f%% | "
              "MMA: tmem-free %.2f%% smem-full %.2f%% | epilogue: tmem-ready %.2f%% read-out %.2f%%\n",
              (long long)m, (long long)n, (long long)p, trace_nt, trace_mc, nmma, trace_maxcl, span / 1e3, 100 * sum[0] / nct / span,
              100 * sum[1] / nct / span, 100 * sum[2] / nmma / span, 100 * sum[3] / nmma / span,
              100 * sum[4] / nct / span, 100 * sum[5] / nct / span);
  }
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, MM_ERR_RUNTIME, "kernel launch failed (m=%lld n=%lld p=%lld dtype=%d): %s", (long long)m,
                   (long long)n, (long long)p, (int)dtype, cudaGetErrorString(e));
  }
  return MM_OK;
}

}  // namespace mmb

using namespace mmb;

static mm_status validate(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, const void* A, const void* B,
                          const void* C) {
  if (!ctx) return MM_ERR_USAGE;
  if (dtype != MM_F64 && dtype != MM_BF16_F32 && dtype != MM_S8_S32 && dtype != MM_F64_EMU)
    return set_err(ctx, MM_ERR_USAGE, "unknown dtype %d", (int)dtype);
  if (m < 1 || n < 1 || p < 1)
    return set_err(ctx, MM_ERR_USAGE, "dimensions must be >= 1: A is %lld x %lld, B is %lld x %lld", (long long)m,
                   (long long)n, (long long)n, (long long)p);
  if (!A || !B || !C) return set_err(ctx, MM_ERR_USAGE, "NULL operand pointer (A=%p B=%p C=%p)", A, B, C);
  // TMA coordinates are int32 and dims < 2^32; tile indices are int.
  const int64_t lim = (int64_t)1 << 31;
  if (m >= lim || n >= lim || p >= lim)
    return set_err(ctx, MM_ERR_UNSUPPORTED, "dimension >= 2^31 (m=%lld n=%lld p=%lld)", (long long)m, (long long)n,
                   (long long)p);
  const size_t ei = dtype_in_size(dtype), eo = dtype_out_size(dtype);
  const __int128 bA = (__int128)m * n * ei, bB = (__int128)n * p * ei, bC = (__int128)m * p * eo;
  const __int128 maxb = ((__int128)1 << 62);
  if (bA > maxb || bB > maxb || bC > maxb) return set_err(ctx, MM_ERR_UNSUPPORTED, "operand byte size overflows int64");
  if (ranges_overlap(C, (size_t)bC, A, (size_t)bA) || ranges_overlap(C, (size_t)bC, B, (size_t)bB))
    return set_err(ctx, MM_ERR_USAGE, "C (%lld x %lld) overlaps A or B", (long long)m, (long long)p);
  return MM_OK;
}

extern "C" {

__attribute__((visibility("default"))) const char* mm_version(void) { return "mm_b200 " MM_VERSION " sm_100a"; }

__attribute__((visibility("default"))) uint64_t mm_launches(const mm_ctx* ctx) { return ctx ? ctx->launches : 0; }

__attribute__((visibility("default"))) const char* mm_status_string(mm_status s) {
  switch (s) {
    case MM_OK: return "MM_OK";
    case MM_ERR_RUNTIME: return "MM_ERR_RUNTIME";
    case MM_ERR_USAGE: return "MM_ERR_USAGE";
    case MM_ERR_UNSUPPORTED: return "MM_ERR_UNSUPPORTED";
    case MM_ERR_WORKSPACE: return "MM_ERR_WORKSPACE";
  }
  return "MM_ERR_UNKNOWN";
}

__attribute__((visibility("default"))) const char* mm_last_error(const mm_ctx* ctx) {
  return ctx ? ctx->last_error.c_str() : "NULL context";
}

__attribute__((visibility("default"))) mm_status mm_create(int device, void* workspace, size_t workspace_bytes,
                                                           mm_ctx** out) {
  if (!out) return MM_ERR_USAGE;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    return MM_ERR_UNSUPPORTED;
  }
  if (device < 0 || device >= ndev) return MM_ERR_USAGE;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return MM_ERR_RUNTIME;
  if (prop.major != 10 || prop.minor != 0) return MM_ERR_UNSUPPORTED;  // sm_100a code only
  mm_ctx* ctx = new mm_ctx();
  ctx->device = device;
  ctx->num_sms = prop.multiProcessorCount;
  ctx->cc_major = prop.major;
  ctx->cc_minor = prop.minor;
  ctx->user_ws = workspace;
  ctx->user_ws_bytes = workspace ? workspace_bytes : 0;
  knobs_refresh();
  if (const char* e = knob("MM_WAVE_SYNC")) ctx->wave_sync = atoi(e);
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(device);
  if (cudaMalloc(&ctx->d_err, 8 * sizeof(int)) != cudaSuccess || cudaMemset(ctx->d_err, 0, 8 * sizeof(int)) != cudaSuccess) {
    cudaSetDevice(prev);
    delete ctx;
    return MM_ERR_RUNTIME;
  }
  cudaSetDevice(prev);
  *out = ctx;
  return MM_OK;
}

__attribute__((visibility("default"))) void mm_destroy(mm_ctx* ctx) {
  if (!ctx) return;
  DeviceGuard dg(ctx->device);
  cudaDeviceSynchronize();
  mm_release_comms(ctx);
  mm_release_ipc(ctx);
  if (ctx->ws) cudaFree(ctx->ws);
  if (ctx->sk_ws) cudaFree(ctx->sk_ws);
  if (ctx->sk_flags) cudaFree(ctx->sk_flags);
  if (ctx->trace_buf) cudaFree(ctx->trace_buf);
  if (ctx->clk_buf) cudaFree(ctx->clk_buf);
  if (ctx->emu_buf) cudaFree(ctx->emu_buf);
  for (auto& b : ctx->hbuf)
    if (b) cudaFree(b);
  for (auto& b : ctx->sbuf)
    if (b) cudaFree(b);
  if (ctx->s_in) cudaStreamDestroy(ctx->s_in);
  if (ctx->s_out) cudaStreamDestroy(ctx->s_out);
  if (ctx->ev_last) cudaEventDestroy(ctx->ev_last);
  if (ctx->d_err) cudaFree(ctx->d_err);
  delete ctx;
}

__attribute__((visibility("default"))) mm_status mm_gemm(mm_ctx* ctx, int64_t m, int64_t n, int64_t p,
                                                         mm_dtype dtype, const void* A, const void* B, void* C,
                                                         void* stream) {
  if (!ctx) return MM_ERR_USAGE;
  knobs_refresh();
  DeviceGuard dg(ctx->device);
  mm_status st = validate(ctx, m, n, p, dtype, A, B, C);
  if (st == MM_OK) st = refuse_diag_knobs(ctx);
  if (st != MM_OK) return st;
  return gemm_ld(ctx, m, n, p, dtype, A, n, B, p, C, p, 0, static_cast<cudaStream_t>(stream));
}

namespace {
// Device scratch one product may need (upper bound; SMs <= kSmBound): zero-padded copies of A and B
// (edge path, as if neither were 16-B pitched), split-tail partial slabs (two slots per CTA) and the
// per-tile tickets + publish counts.
constexpr int64_t kSmBound = 160;
int64_t product_scratch(int64_t m, int64_t n, int64_t p, mm_dtype dt) {
  const int64_t ei = (int64_t)dtype_in_size(dt), al = 16 / ei;
  const int64_t pad = round_up(m * round_up(n, al) * ei, 256) + round_up(n * round_up(p, al) * ei, 256);
  int64_t slabs, flags;
  if (dt == MM_F64) {  // 128x128 tiles at most; tiles >= 32x32
    slabs = kSmBound * 2 * 128 * 128 * 8;
    flags = 2 * ((m + 31) / 32) * ((p + 31) / 32) * 4;
  } else {  // CTA slabs of 128 x 512 words at most; tiles >= 128 x 256 per CTA
    slabs = kSmBound * 2 * 128 * 512 * 4;
    flags = 2 * ((m + 127) / 128) * ((p + 255) / 256) * 4 * 2;
  }
  return pad + round_up(slabs, 256) + round_up(std::max<int64_t>(flags, 256), 256);
}
// MM_F64_EMU: residue planes + the batched INT8 product's own scratch (N planes of whole 256-row tiles)
int64_t emu_or_product_scratch(int64_t m, int64_t n, int64_t p, mm_dtype dt) {
  if (dt != MM_F64_EMU) return product_scratch(m, n, p, dt);
  const int64_t nmod = f64_emu_moduli(n, nullptr, nullptr);
  return (int64_t)f64_emu_scratch(m, n, p) + product_scratch(nmod * ((m + 255) / 256 * 256), (n + 15) / 16 * 16, p, MM_S8_S32);
}
}  // namespace

__attribute__((visibility("default"))) mm_status mm_f64_emu_plan(int64_t n, int* moduli, int* count, int* beta) {
  if (n < 1 || !count || !beta) return MM_ERR_USAGE;
  if (n > f64_emu_max_n()) return MM_ERR_UNSUPPORTED;
  int mods[16];
  const int c = f64_emu_moduli(n, beta, mods);
  if (c == 0) return MM_ERR_UNSUPPORTED;
  *count = c;
  if (moduli)
    for (int l = 0; l < c; ++l) moduli[l] = mods[l];
  return MM_OK;
}

__attribute__((visibility("default"))) size_t mm_workspace_size(int64_t m, int64_t n, int64_t p, mm_dtype dtype,
                                                                 mm_layout layout, int G) {
  if (m < 1 || n < 1 || p < 1 || G < 1) return 0;
  if (dtype != MM_F64 && dtype != MM_BF16_F32 && dtype != MM_S8_S32 && dtype != MM_F64_EMU) return 0;
  if (dtype == MM_F64_EMU && n > f64_emu_max_n()) return 0;
  if (layout != MM_ROW_BLOCK && layout != MM_SUMMA_2D && layout != MM_SUMMA_25D) return 0;
  if (layout != MM_ROW_BLOCK && dtype != MM_F64 && dtype != MM_F64_EMU) return 0;
  knobs_refresh();
  int64_t best = 0;
  auto consider = [&](int pr, int pc, unsigned flags) {
    for (int r = 0; r < G; ++r) {
      mm_plan_info info;
      std::vector<mm_plan_step> steps;
      if (mm_shard_plan(m, n, p, dtype, layout, pr, pc, flags, 0, G, r, 0, nullptr, 0, &info) != MM_OK) continue;
      steps.resize((size_t)info.steps);
      mm_shard_plan(m, n, p, dtype, layout, pr, pc, flags, 0, G, r, 0, steps.data(), info.steps, &info);
      int64_t total = 512;  // IPC exchange word + barrier word
      for (int i = 0; i < 4; ++i) total += round_up(std::max<int64_t>(info.stage_bytes[i], 0), 256);
      int64_t g = 0;
      for (const mm_plan_step& s : steps)
        if (s.op == MM_OP_GEMM) g = std::max(g, emu_or_product_scratch(s.m, s.n, s.p, dtype));
      best = std::max(best, total + g);
      if (G == 1) break;
    }
  };
  if (G == 1 && layout == MM_ROW_BLOCK) return (size_t)emu_or_product_scratch(m, n, p, dtype);
  if (layout == MM_ROW_BLOCK) {
    consider(0, 0, MM_BCAST_B);  // staging buffers of the broadcast (the largest variant)
    consider(0, 0, 0);
  } else {
    for (int pr = 1; pr <= G; ++pr) {
      if (G % pr) continue;
      const int rest = G / pr;
      for (int pc = 1; pc <= rest; ++pc) {
        if (rest % pc) continue;
        if (layout == MM_SUMMA_2D && pr * pc != G) continue;
        consider(pr, pc, layout == MM_SUMMA_25D ? (unsigned)MM_REPLICATE : 0u);
      }
    }
  }
  return (size_t)best;
}

__attribute__((visibility("default"))) mm_status mm_clock_meter(mm_ctx* ctx, int enable, double* mhz) {
  if (!ctx) return MM_ERR_USAGE;
  DeviceGuard dg(ctx->device);
  const size_t bytes = 4096 * 4 * sizeof(unsigned long long);
  if (enable) {
    if (!ctx->clk_buf && cudaMalloc(&ctx->clk_buf, bytes) != cudaSuccess) {
      cudaGetLastError();
      ctx->clk_buf = nullptr;
      return set_err(ctx, MM_ERR_WORKSPACE, "clock meter buffer allocation failed");
    }
    if (cudaMemset(ctx->clk_buf, 0, bytes) != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "clock meter reset failed");
    ctx->clk_on = true;
    if (mhz) *mhz = 0.0;
    return MM_OK;
  }
  ctx->clk_on = false;
  if (mhz) *mhz = 0.0;
  if (!ctx->clk_buf) return MM_OK;
  if (cudaDeviceSynchronize() != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "clock meter: synchronisation failed");
  std::vector<unsigned long long> h(4096 * 4);
  if (cudaMemcpy(h.data(), ctx->clk_buf, bytes, cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "clock meter: read-back failed");
  double cyc = 0, ns = 0;
  for (int c = 0; c < 4096; ++c) {
    const unsigned long long* r = &h[(size_t)c * 4];
    if (r[3] > r[1] && r[2] > r[0]) {
      cyc += (double)(r[2] - r[0]);
      ns += (double)(r[3] - r[1]);
    }
  }
  if (mhz) *mhz = ns > 0 ? 1e3 * cyc / ns : 0.0;
  return MM_OK;
}

__attribute__((visibility("default"))) mm_status mm_sync_check(mm_ctx* ctx, void* stream) {
  if (!ctx) return MM_ERR_USAGE;
  DeviceGuard dg(ctx->device);
  cudaError_t e = cudaStreamSynchronize(static_cast<cudaStream_t>(stream));
  if (e != cudaSuccess) return set_err(ctx, MM_ERR_RUNTIME, "stream sync failed: %s", cudaGetErrorString(e));
  int h = 0;
  if (cudaMemcpy(&h, ctx->d_err, sizeof(int), cudaMemcpyDeviceToHost) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "reading the device error word failed");
  if (h != 0) {
    cudaMemset(ctx->d_err, 0, 8 * sizeof(int));  // error word + wave-barrier / pacing counters
    if (ctx->sk_flags) cudaMemset(ctx->sk_flags, 0, ctx->sk_flag_count * sizeof(unsigned));
    if (h == kErrNonFinite)
      return set_err(ctx, MM_ERR_RUNTIME, "MM_F64_EMU: an operand holds Inf or NaN (the emulation needs finite "
                                          "inputs; C is undefined — use MM_F64 for IEEE propagation)");
    return set_err(ctx, MM_ERR_RUNTIME, "device pipeline wait timed out (code %d)", h);
  }
  return MM_OK;
}

// Host operands.  PCIe, not the tensor cores, bounds this call (C4: 1 GiB in,
// 1 GiB out vs 7 ms of math), so the copies are scheduled to keep both PCIe
// directions busy: A arrives in row blocks A_i and B in column panels B_j,
// interleaved A_0, B_0, A_1, B_1, ... (the computable part of C grows as a
// square), each block C_ij = A_i·B_j is computed as soon as both have landed
// and copied back while later blocks are still coming in.  Streams: s_in
// (H2D), the caller's stream (products), s_out (D2H); events order them.
__attribute__((visibility("default"))) mm_status mm_gemm_host(mm_ctx* ctx, int64_t m, int64_t n, int64_t p,
                                                              mm_dtype dtype, const void* A, const void* B, void* C,
                                                              void* stream) {
  if (!ctx) return MM_ERR_USAGE;
  knobs_refresh();
  DeviceGuard dg(ctx->device);
  mm_status st = validate(ctx, m, n, p, dtype, A, B, C);
  if (st == MM_OK) st = refuse_diag_knobs(ctx);
  if (st != MM_OK) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t ei = dtype_in_size(dtype), eo = dtype_out_size(dtype);
  if (!ctx->s_in) {
    if (cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&ctx->s_out, cudaStreamNonBlocking) != cudaSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "stream creation failed");
  }
  if ((st = ensure_buffer(ctx, &ctx->hbuf[0], &ctx->hbuf_bytes[0], (size_t)(m * n) * ei)) != MM_OK) return st;
  if ((st = ensure_buffer(ctx, &ctx->hbuf[1], &ctx->hbuf_bytes[1], (size_t)(n * p) * ei)) != MM_OK) return st;
  if ((st = ensure_buffer(ctx, &ctx->hbuf[2], &ctx->hbuf_bytes[2], (size_t)(m * p) * eo)) != MM_OK) return st;
  uint8_t* dA = static_cast<uint8_t*>(ctx->hbuf[0]);
  uint8_t* dB = static_cast<uint8_t*>(ctx->hbuf[1]);
  uint8_t* dC = static_cast<uint8_t*>(ctx->hbuf[2]);
  const uint8_t* hA = static_cast<const uint8_t*>(A);
  const uint8_t* hB = static_cast<const uint8_t*>(B);
  uint8_t* hC = static_cast<uint8_t*>(C);

  // ~8 blocks per axis, multiples of 256 (one CTA-pair tile); small problems: one block.
  const int64_t small = (int64_t)64 << 20;
  const bool tiny = (double)(m * n + n * p) * ei < (double)small;
  int64_t nblk = 4;  // measured best for C4 (tools/e2e_probe.py: 28.6 ms vs 31.5 ms at 8)
  if (const char* env = knob("MM_HOST_BLOCKS")) nblk = std::max<int64_t>(1, atoll(env));  // tuning knob
  const int64_t rb = tiny ? m : std::min(m, round_up((m + nblk - 1) / nblk, 256));
  const int64_t cb = tiny ? p : std::min(p, round_up((p + nblk - 1) / nblk, 256));
  const int I = (int)((m + rb - 1) / rb), J = (int)((p + cb - 1) / cb);
  std::vector<cudaEvent_t> evA(I), evB(J), evC((size_t)I * J);
  cudaEvent_t evStart;
#ifdef MM_DIAG
  const bool trace = knob("MM_HOST_TRACE") != nullptr;  // debug: print the copy/compute timeline
#else
  const bool trace = false;
#endif
  const unsigned evflags = trace ? cudaEventDefault : cudaEventDisableTiming;
  std::vector<cudaEvent_t> evD((size_t)I * J);
  cudaEventCreateWithFlags(&evStart, evflags);
  for (auto& e : evA) cudaEventCreateWithFlags(&e, evflags);
  for (auto& e : evB) cudaEventCreateWithFlags(&e, evflags);
  for (auto& e : evC) cudaEventCreateWithFlags(&e, evflags);
  for (auto& e : evD) cudaEventCreateWithFlags(&e, evflags);
  // copies must not overtake earlier work on the caller's stream that uses the staging buffers
  cudaEventRecord(evStart, s);
  cudaStreamWaitEvent(ctx->s_in, evStart, 0);
  cudaStreamWaitEvent(ctx->s_out, evStart, 0);

  cudaError_t e = cudaSuccess;
  int ia = 0, jb = 0;  // A row blocks / B column panels issued so far
  auto compute = [&](int i, int j) {
    const int64_t r0 = (int64_t)i * rb, rows = std::min(rb, m - r0);
    const int64_t c0 = (int64_t)j * cb, cols = std::min(cb, p - c0);
    cudaStreamWaitEvent(s, evA[i], 0);
    cudaStreamWaitEvent(s, evB[j], 0);
    if (st == MM_OK)
      st = gemm_ld(ctx, rows, n, cols, dtype, dA + r0 * n * ei, n, dB + c0 * ei, p, dC + (r0 * p + c0) * eo, p, 0, s);
    cudaEventRecord(evC[(size_t)i * J + j], s);
    cudaStreamWaitEvent(ctx->s_out, evC[(size_t)i * J + j], 0);
    if (e == cudaSuccess)
      e = cudaMemcpy2DAsync(hC + (r0 * p + c0) * eo, (size_t)p * eo, dC + (r0 * p + c0) * eo, (size_t)p * eo,
                            (size_t)cols * eo, (size_t)rows, cudaMemcpyDeviceToHost, ctx->s_out);
    cudaEventRecord(evD[(size_t)i * J + j], ctx->s_out);
  };
  while ((ia < I || jb < J) && e == cudaSuccess && st == MM_OK) {
    const bool takeA = ia < I && (ia <= jb || jb == J);
    if (takeA) {
      const int64_t r0 = (int64_t)ia * rb, rows = std::min(rb, m - r0);
      e = cudaMemcpyAsync(dA + r0 * n * ei, hA + r0 * n * ei, (size_t)(rows * n) * ei, cudaMemcpyHostToDevice,
                          ctx->s_in);
      cudaEventRecord(evA[ia], ctx->s_in);
      for (int j = 0; j < jb; ++j) compute(ia, j);
      ++ia;
    } else {
      const int64_t c0 = (int64_t)jb * cb, cols = std::min(cb, p - c0);
      e = cudaMemcpy2DAsync(dB + c0 * ei, (size_t)p * ei, hB + c0 * ei, (size_t)p * ei, (size_t)cols * ei, (size_t)n,
                            cudaMemcpyHostToDevice, ctx->s_in);
      cudaEventRecord(evB[jb], ctx->s_in);
      for (int i = 0; i < ia; ++i) compute(i, jb);
      ++jb;
    }
  }
  cudaError_t e2 = cudaStreamSynchronize(ctx->s_out);
  cudaError_t e3 = cudaStreamSynchronize(s);
  cudaStreamSynchronize(ctx->s_in);
  if (trace) {
    auto ms = [&](cudaEvent_t ev) { float t = 0; cudaEventElapsedTime(&t, evStart, ev); return t; };
    for (int i = 0; i < I; ++i) fprintf(stderr, "[mm_gemm_host] A%d in  %8.3f ms\n", i, ms(evA[i]));
    for (int j = 0; j < J; ++j) fprintf(stderr, "[mm_gemm_host] B%d in  %8.3f ms\n", j, ms(evB[j]));
    for (int i = 0; i < I; ++i)
      for (int j = 0; j < J; ++j)
        fprintf(stderr, "[mm_gemm_host] C%d,%d done %8.3f ms  out %8.3f ms\n", i, j, ms(evC[(size_t)i * J + j]),
                ms(evD[(size_t)i * J + j]));
  }
  cudaEventDestroy(evStart);
  for (auto& x : evD) cudaEventDestroy(x);
  for (auto& x : evA) cudaEventDestroy(x);
  for (auto& x : evB) cudaEventDestroy(x);
  for (auto& x : evC) cudaEventDestroy(x);
  if (st != MM_OK) return st;
  if (e != cudaSuccess || e2 != cudaSuccess || e3 != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "host pipeline failed: %s",
                   cudaGetErrorString(e != cudaSuccess ? e : (e2 != cudaSuccess ? e2 : e3)));
  return mm_sync_check(ctx, s);
}

}  // extern "C"
