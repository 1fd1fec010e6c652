// ctx.h — the mm_ctx object and internal helpers shared by the ABI translation units.
#pragma once
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>
#include <vector>

#include "mm.h"

struct mm_ctx {
  int device = 0;
  int num_sms = 0;
  int cc_major = 0, cc_minor = 0;
  void* user_ws = nullptr;
  size_t user_ws_bytes = 0;
  int c_remote = 0;  // set around products whose C is a peer GPU's memory (fused row-block gather)
  int sm_reserve = 0;  // SMs left free for concurrent (communication) kernels, set around overlapped products
  // cross-stream ordering of the context's scratch (wave counters, split-tile counters and slabs,
  // padding buffer): a product on a stream other than the previous one waits for the previous one
  cudaStream_t last_stream = nullptr;
  cudaEvent_t ev_last = nullptr;
  bool ev_last_valid = false;
  void* ws = nullptr;  // internal, grow-only (padding path)
  size_t ws_bytes = 0;
  int* d_err = nullptr;  // [0] device error word (pipeline timeouts), [1..4] wave-barrier / pacing counters, abandoned flag
  int wave_sync = 1;
  // mm_gemm_host staging
  void* hbuf[3] = {nullptr, nullptr, nullptr};
  size_t hbuf_bytes[3] = {0, 0, 0};
  cudaStream_t s_in = nullptr, s_out = nullptr;
  // sharded scratch (panels, gathered rows)
  void* sbuf[4] = {nullptr, nullptr, nullptr, nullptr};
  size_t sbuf_bytes[4] = {0, 0, 0, 0};
  // sharded plans: ROW / COL / DEPTH sub-communicators (ncclComm_t, index = mm_plan_comm), cached
  // per (parent communicator, split colour, key)
  void* sub_comm[4] = {nullptr, nullptr, nullptr, nullptr};
  void* split_parent = nullptr;
  int64_t split_sig[4] = {-1, -1, -1, -1};  // (layout, grid_rows, grid_cols, G): the same on every rank
  std::vector<cudaEvent_t> plan_events;  // the plan's event ids
  void* sk_ws = nullptr;  // stream-K partial tiles (both kernels)
  size_t sk_ws_bytes = 0;
  unsigned* sk_flags = nullptr;  // stream-K per-tile counters (self-resetting)
  size_t sk_flag_count = 0;
  void* ipc_xchg = nullptr;  // device staging for the IPC handle exchange (fused gather)
  struct IpcMap {
    std::string handle;  // cudaIpcMemHandle_t bytes
    void* base;
    size_t bytes;
  };
  std::vector<IpcMap> ipc_open;  // allocations of other processes mapped by mm_ipc_open
  struct Window {  // mm_window_alloc: NCCL symmetric memory of this rank
    void* base;
    size_t bytes;
    void* win;   // ncclWindow_t
    void* comm;  // ncclComm_t it is registered with
  };
  std::vector<Window> windows;
  void* emu_buf = nullptr;    // MM_F64_EMU: residue planes of A, B and C, exponents
  size_t emu_bytes = 0;
  int res_mod = 0;  // MM_F64_EMU: its INT8 products store C mod res_mod as bytes (0 = INT32 C)
  int res_nbat = 0;  // > 1: one launch for res_nbat batches stacked along M (moduli res_mods[b])
  int res_mods[16] = {};
  int64_t res_bat_rows = 0, res_bat_krows = 0;  // rows per batch of A / C and of B
  void* bar_buf = nullptr;   // one int for the communicator barrier
  void* trace_buf = nullptr;  // MM_TRACE per-CTA counters
  unsigned long long* clk_buf = nullptr;  // clock meter: 4096 CTAs x {c0, t0, c1, t1} of the last launch
  bool clk_on = false;
  uint64_t launches = 0;  // kernels launched by this context
  // encoded tensor maps of recent calls (host cost of cuTensorMapEncodeTiled per call), keyed by
  // everything the encoding depends on; round-robin replacement
  struct MapEntry {
    uint64_t key[8];
    CUtensorMap map;
  };
  MapEntry map_cache[32] = {};
  int map_cache_used = 0, map_cache_next = 0;
  std::string last_error;
};

extern "C" void mm_release_comms(mm_ctx* ctx);  // shard.cu: sub-communicators
extern "C" void mm_release_ipc(mm_ctx* ctx);    // shard.cu: IPC mappings, events, small buffers

namespace mmb {

// Makes the context's device current for the duration of an ABI call (the caller's current
// device may differ: operands, stream and context belong to ctx->device).
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) { cudaGetLastError(); prev = -1; }
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    int cur = -1;
    cudaGetDevice(&cur);
    if (prev >= 0 && cur != prev) cudaSetDevice(prev);
  }
};

mm_status set_err(mm_ctx* ctx, mm_status s, const char* fmt, ...);
size_t dtype_in_size(mm_dtype t);
size_t dtype_out_size(mm_dtype t);
// grow-only device buffer owned by ctx (synchronizes the device before freeing an old buffer)
mm_status ensure_buffer(mm_ctx* ctx, void** buf, size_t* have, size_t need);
// internal C (+)= A·B with explicit leading dimensions (elements); beta_one only for MM_F64.
// MM_OK, or MM_ERR_UNSUPPORTED when a diagnostic-only knob is set for the release library.
mm_status refuse_diag_knobs(mm_ctx* ctx);
mm_status gemm_ld(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, const void* A, int64_t lda,
                  const void* B, int64_t ldb, void* C, int64_t ldc, int beta_one, cudaStream_t s);
// MM_F64_EMU (f64_emu.cu): binary64 product on the INT8 tensor cores (integer scaling, residues modulo
// N coprime moduli, N exact INT8 products, Chinese remaindering)
mm_status gemm_f64_emu(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, const double* A, int64_t lda, const double* B,
                       int64_t ldb, double* C, int64_t ldc, int beta_one, cudaStream_t s);
size_t f64_emu_scratch(int64_t m, int64_t n, int64_t p);
int64_t f64_emu_max_n();
// moduli count N (0: none) and β for inner dimension n; the moduli themselves into mods (room for 16)
int f64_emu_moduli(int64_t n, int* beta, int* mods);

}  // namespace mmb
