// shard.cu — multi-GPU products, one process per GPU, NCCL over NVLink/NVSwitch.
//
// The paper parallelises the product across threads by splitting the outer
// (row) loop (§III-B1) and discusses process-level
// distribution with SUMMA (§III-B2).  Two layouts:
//
//   MM_ROW_BLOCK — rank r owns a contiguous block of rows of A and C
//     (mm_shard_range, SPEC.md:210 ⌈m/G⌉ rule); B is replicated
//     (optionally broadcast from `root` first); C optionally gathered —
//     by NCCL send/recv after the product (MM_GATHER_C), or fused into the
//     product (MM_GATHER_C_FUSED): each rank's tcgen05/DMMA kernel stores its C
//     tiles straight into the root's C_full through a CUDA-IPC peer mapping
//     (TMA stores over NVLink), so the gather overlaps the math tile by tile.
//     No exchange is needed for the product itself.
//   MM_SUMMA_2D — ranks form a grid; for each k-panel the owner column of
//     A broadcasts its panel along its grid row and the owner row of B along
//     its grid column; every rank accumulates C_ij += A_i,panel · B_panel,j.
//     Panels are double-buffered: the broadcasts of panel t+1 (comm stream)
//     overlap the local product of panel t (caller's stream).
//
// NCCL symbols are resolved at run time from the libnccl.so.2 already loaded
// in the process (the one torch uses), so the library never links a second,
// mismatched NCCL.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <cstdlib>
#include <mutex>
#include <vector>

#include "ctx.h"
#include "kernels.h"
#include "knobs.h"
#include <nccl_device.h>  // ncclGetPeerPointer (header-only device helper over a registered window)

namespace mmb {
namespace {

struct NcclApi {
  ncclResult_t (*Broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, int, ncclComm_t, cudaStream_t) =
      nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*CommSplit)(ncclComm_t, int, int, ncclComm_t*, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*CommCount)(const ncclComm_t, int*) = nullptr;
  ncclResult_t (*CommUserRank)(const ncclComm_t, int*) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  // symmetric memory (NCCL >= 2.27; optional: MM_C_WINDOW needs them)
  ncclResult_t (*MemAlloc)(void**, size_t) = nullptr;
  ncclResult_t (*MemFree)(void*) = nullptr;
  ncclResult_t (*CommWindowRegister)(ncclComm_t, void*, size_t, ncclWindow_t*, int) = nullptr;
  ncclResult_t (*CommWindowDeregister)(ncclComm_t, ncclWindow_t) = nullptr;
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi& nccl_api() {
  std::call_once(g_nccl_once, [] {
    // MM_NCCL_LIB (explicit override, e.g. the test suite's one-GPU shim) first, else the
    // libnccl.so.2 torch already loaded
    void* h = nullptr;
    if (const char* p = getenv("MM_NCCL_LIB")) h = dlopen(p, RTLD_LAZY | RTLD_LOCAL);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOLOAD | RTLD_LAZY);
    if (!h) return;
#define LOAD(field, name) g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name))
    LOAD(Broadcast, "ncclBroadcast");
    LOAD(Send, "ncclSend");
    LOAD(Recv, "ncclRecv");
    LOAD(AllReduce, "ncclAllReduce");
    LOAD(Reduce, "ncclReduce");
    LOAD(GroupStart, "ncclGroupStart");
    LOAD(GroupEnd, "ncclGroupEnd");
    LOAD(CommSplit, "ncclCommSplit");
    LOAD(CommDestroy, "ncclCommDestroy");
    LOAD(CommCount, "ncclCommCount");
    LOAD(CommUserRank, "ncclCommUserRank");
    LOAD(GetErrorString, "ncclGetErrorString");
    LOAD(MemAlloc, "ncclMemAlloc");
    LOAD(MemFree, "ncclMemFree");
    LOAD(CommWindowRegister, "ncclCommWindowRegister");
    LOAD(CommWindowDeregister, "ncclCommWindowDeregister");
#undef LOAD
    g_nccl.ok = g_nccl.Broadcast && g_nccl.AllReduce && g_nccl.Reduce && g_nccl.Send && g_nccl.Recv && g_nccl.GroupStart && g_nccl.GroupEnd &&
                g_nccl.CommSplit && g_nccl.CommCount && g_nccl.CommUserRank && g_nccl.GetErrorString;
  });
  return g_nccl;
}

#define NCCL_CHECK(ctx, call)                                                                               \
  do {                                                                                                      \
    ncclResult_t _r = (call);                                                                               \
    if (_r != ncclSuccess)                                                                                  \
      return set_err(ctx, MM_ERR_RUNTIME, "%s failed: %s", #call, nccl_api().GetErrorString(_r));               \
  } while (0)

// cuMemGetAddressRange from the driver (base + size of the allocation holding a pointer).
typedef CUresult (*GetAddrRangeFn)(CUdeviceptr*, size_t*, CUdeviceptr);
GetAddrRangeFn addr_range_fn() {
  static GetAddrRangeFn fn = [] {
    void* f = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &f, 12000, cudaEnableDefault, &q) != cudaSuccess ||
        q != cudaDriverEntryPointSuccess) {
      cudaGetLastError();
      return (GetAddrRangeFn) nullptr;
    }
    return reinterpret_cast<GetAddrRangeFn>(f);
  }();
  return fn;
}

// Collective: every rank learns a pointer to the root's `root_ptr` it can store to (the root's own
// pointer on the root; elsewhere a CUDA-IPC mapping of the root's allocation — over NVLink when the
// root is another GPU).  The handle (mm_ipc_export) travels by ncclBroadcast.
mm_status peer_pointer_of_root(mm_ctx* ctx, void* root_ptr, int root, int r, ncclComm_t comm, cudaStream_t s,
                               uint8_t** out) {
  mm_ipc_handle msg;
  memset(&msg, 0, sizeof msg);
  if (r == root) {
    mm_status st = mm_ipc_export(ctx, root_ptr, &msg);
    if (st != MM_OK) return st;
  }
  if (!ctx->ipc_xchg && cudaMalloc(&ctx->ipc_xchg, 256) != cudaSuccess)
    return set_err(ctx, MM_ERR_WORKSPACE, "IPC exchange buffer allocation failed");
  if (r == root && cudaMemcpyAsync(ctx->ipc_xchg, &msg, sizeof msg, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "IPC handle staging failed");
  NCCL_CHECK(ctx, nccl_api().Broadcast(ctx->ipc_xchg, ctx->ipc_xchg, sizeof msg, ncclUint8, root, comm, s));
  if (cudaMemcpyAsync(&msg, ctx->ipc_xchg, sizeof msg, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "IPC handle exchange failed");
  if (r == root) {
    *out = static_cast<uint8_t*>(root_ptr);
    return MM_OK;
  }
  void* p = nullptr;
  mm_status st = mm_ipc_open(ctx, &msg, &p);
  if (st != MM_OK) return st;
  *out = static_cast<uint8_t*>(p);
  return MM_OK;
}

// The root's address of a symmetric buffer: NCCL maps every rank's window of a node into one flat
// range of this process (LSA, over NVLink); ncclGetPeerPointer reads the window's device-side
// descriptor, so it runs on the device.
__global__ void window_peer_ptr_kernel(ncclWindow_t w, size_t off, int peer, void** out) {
  *out = ncclGetPeerPointer(w, off, peer);
}

// MM_C_WINDOW: every rank's C_full lies in a window of this context at the same offset; the root's
// copy is at ncclGetPeerPointer(window, offset, root).  Local, no communication.
mm_status window_pointer_of_root(mm_ctx* ctx, void* my_ptr, int root, cudaStream_t s, uint8_t** out) {
  const mm_ctx::Window* w = nullptr;
  for (const auto& e : ctx->windows)
    if (static_cast<uint8_t*>(my_ptr) >= static_cast<uint8_t*>(e.base) &&
        static_cast<uint8_t*>(my_ptr) < static_cast<uint8_t*>(e.base) + e.bytes)
      w = &e;
  if (!w) return set_err(ctx, MM_ERR_USAGE, "MM_C_WINDOW: C_full %p is not in a buffer from mm_window_alloc", my_ptr);
  const size_t off = static_cast<size_t>(static_cast<uint8_t*>(my_ptr) - static_cast<uint8_t*>(w->base));
  if (!ctx->ipc_xchg && cudaMalloc(&ctx->ipc_xchg, 256) != cudaSuccess)
    return set_err(ctx, MM_ERR_WORKSPACE, "window pointer staging allocation failed");
  window_peer_ptr_kernel<<<1, 1, 0, s>>>(static_cast<ncclWindow_t>(w->win), off, root, static_cast<void**>(ctx->ipc_xchg));
  void* p = nullptr;
  if (cudaGetLastError() != cudaSuccess || cudaMemcpyAsync(&p, ctx->ipc_xchg, sizeof p, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess || !p)
    return set_err(ctx, MM_ERR_RUNTIME, "MM_C_WINDOW: resolving the root's window address failed");
  *out = static_cast<uint8_t*>(p);
  return MM_OK;
}

// The executor's view of a plan's buffers.
struct PlanBufs {
  bool c_window = false;  // MM_C_WINDOW: the fused gather's peer address comes from an NCCL window
  uint8_t* p[10] = {};
  const char* name(int b) const {
    static const char* n[10] = {"-", "A_local", "B_local", "C_local", "C_full", "C_peer", "S0", "S1", "S2", "S3"};
    return (b >= 0 && b < 10) ? n[b] : "?";
  }
};

// Sub-communicators of the plan (ROW / COL / DEPTH), split from WORLD with the plan's colours and
// keys and cached in the context.  ncclCommSplit is collective, so whether to (re-)split must be
// decided identically on every rank: the cache key is (parent, layout, grid, G) — the collective's
// arguments — never a rank's own colour or key (two grids can give one rank the same colours and
// another different ones; keying on colours made only some ranks re-split and deadlocked G > 1,
// found by tests/test_gpu_shim_multirank.py).
mm_status plan_comms(mm_ctx* ctx, ncclComm_t world, const mm_plan_info& info, const int64_t sig[4],
                     ncclComm_t comms[4]) {
  const NcclApi& api = nccl_api();
  comms[MM_COMM_WORLD] = world;
  bool same = ctx->split_parent == world;
  for (int i = 0; i < 4; ++i) same = same && ctx->split_sig[i] == sig[i];
  if (!same) {
    mm_release_comms(ctx);
    for (int c = 1; c < 4; ++c) {
      ncclComm_t sub = nullptr;
      if (info.color[c] >= 0) NCCL_CHECK(ctx, api.CommSplit(world, info.color[c], info.key[c], &sub, nullptr));
      ctx->sub_comm[c] = sub;
    }
    for (int i = 0; i < 4; ++i) ctx->split_sig[i] = sig[i];
    ctx->split_parent = world;
  }
  for (int c = 1; c < 4; ++c) comms[c] = static_cast<ncclComm_t>(ctx->sub_comm[c]);
  return MM_OK;
}

// Run rank r's plan: products on the caller's stream (0), communication and staging copies on the
// context's communication stream (1), ordered by the plan's events.
mm_status execute_plan(mm_ctx* ctx, const std::vector<mm_plan_step>& steps, const mm_plan_info& info, PlanBufs& B,
                       mm_dtype dtype, ncclComm_t world, int r, const int64_t split_sig[4], cudaStream_t s0) {
  const NcclApi& api = nccl_api();
  // buffers every step needs must exist (usage errors before anything is enqueued)
  for (const mm_plan_step& st : steps) {
    const int need[3] = {st.dst, st.src, st.src2};
    for (int b : need)
      if (b != MM_BUF_NONE && b != MM_BUF_CPEER && b < MM_BUF_S0 && !B.p[b])
        return set_err(ctx, MM_ERR_USAGE, "rank %d: the sharded plan needs %s (NULL was passed)", r, B.name(b));
  }
  mm_status ss;
  for (int i = 0; i < 4; ++i)
    if (info.stage_bytes[i] > 0) {
      if ((ss = ensure_buffer(ctx, &ctx->sbuf[i], &ctx->sbuf_bytes[i], (size_t)info.stage_bytes[i])) != MM_OK) return ss;
      B.p[MM_BUF_S0 + i] = static_cast<uint8_t*>(ctx->sbuf[i]);
    }
  ncclComm_t comms[4];
  if ((ss = plan_comms(ctx, world, info, split_sig, comms)) != MM_OK) return ss;
  if (!ctx->s_in && cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "stream creation failed");
  cudaStream_t strm[2] = {s0, ctx->s_in};
  while ((int)ctx->plan_events.size() < info.events) {
    cudaEvent_t e;
    if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "event creation failed");
    ctx->plan_events.push_back(e);
  }
  int reserve = 16;  // SMs left to NCCL's kernels while a product overlaps communication
  if (const char* e = knob("MM_COMM_SM_RESERVE")) reserve = std::max(0, atoi(e));  // tuning knob
  struct Restore {  // per-product context state, reset on every exit path
    mm_ctx* c;
    ~Restore() { c->c_remote = 0; c->sm_reserve = 0; }
  } restore{ctx};
  auto at = [&](int b, int64_t off) { return B.p[b] + off; };
  for (size_t i = 0; i < steps.size(); ++i) {
    const mm_plan_step& st = steps[i];
    cudaStream_t sx = strm[st.stream ? 1 : 0];
    cudaError_t ce = cudaSuccess;
    ncclResult_t nr = ncclSuccess;
    switch (st.op) {
      case MM_OP_GEMM: {
        ctx->c_remote = st.dst == MM_BUF_CPEER ? 1 : 0;  // C in a peer's memory: plain stores only
        ctx->sm_reserve = st.overlap ? reserve : 0;
        mm_status g = gemm_ld(ctx, st.m, st.n, st.p, dtype, at(st.src, st.src_off), st.src_ld, at(st.src2, st.src2_off),
                              st.src2_ld, at(st.dst, st.dst_off), st.dst_ld, st.beta, sx);
        ctx->c_remote = 0;
        ctx->sm_reserve = 0;
        if (g != MM_OK) return g;
        break;
      }
      case MM_OP_COPY2D:
        ce = cudaMemcpy2DAsync(at(st.dst, st.dst_off), (size_t)st.dst_ld, at(st.src, st.src_off), (size_t)st.src_ld,
                               (size_t)st.n, (size_t)st.m, cudaMemcpyDeviceToDevice, sx);
        break;
      case MM_OP_BCAST:
        nr = api.Broadcast(at(st.dst, st.dst_off), at(st.dst, st.dst_off), (size_t)st.n, ncclUint8, st.peer,
                           comms[st.comm], sx);
        break;
      case MM_OP_SEND:
        nr = api.Send(at(st.src, st.src_off), (size_t)st.n, ncclUint8, st.peer, comms[st.comm], sx);
        break;
      case MM_OP_RECV:
        nr = api.Recv(at(st.dst, st.dst_off), (size_t)st.n, ncclUint8, st.peer, comms[st.comm], sx);
        break;
      case MM_OP_GROUP_START: nr = api.GroupStart(); break;
      case MM_OP_GROUP_END: nr = api.GroupEnd(); break;
      case MM_OP_REDUCE_SUM:
        nr = api.Reduce(at(st.dst, st.dst_off), at(st.dst, st.dst_off), (size_t)st.n, ncclFloat64, ncclSum, st.peer,
                        comms[st.comm], sx);
        break;
      case MM_OP_MEMSET0: ce = cudaMemsetAsync(at(st.dst, st.dst_off), 0, (size_t)st.n, sx); break;
      case MM_OP_BARRIER:
        if (!ctx->bar_buf && cudaMalloc(&ctx->bar_buf, 16) != cudaSuccess)
          return set_err(ctx, MM_ERR_WORKSPACE, "barrier buffer allocation failed");
        nr = api.AllReduce(ctx->bar_buf, ctx->bar_buf, 1, ncclInt32, ncclSum, comms[st.comm], sx);
        break;
      case MM_OP_MAP_PEER: {
        uint8_t* peer = nullptr;
        mm_status g = B.c_window ? window_pointer_of_root(ctx, B.p[MM_BUF_CFULL], st.peer, sx, &peer)
                                 : peer_pointer_of_root(ctx, B.p[MM_BUF_CFULL], st.peer, r, world, sx, &peer);
        if (g != MM_OK) return g;
        B.p[MM_BUF_CPEER] = peer;
        break;
      }
      case MM_OP_RECORD: ce = cudaEventRecord(ctx->plan_events[st.event], sx); break;
      case MM_OP_WAIT: ce = cudaStreamWaitEvent(sx, ctx->plan_events[st.event], 0); break;
      default: return set_err(ctx, MM_ERR_RUNTIME, "unknown plan step %d", st.op);
    }
    if (ce != cudaSuccess) {
      cudaGetLastError();
      return set_err(ctx, MM_ERR_RUNTIME, "rank %d plan step %zu (op %d) failed: %s", r, i, st.op,
                     cudaGetErrorString(ce));
    }
    if (nr != ncclSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "rank %d plan step %zu (op %d) NCCL failure: %s", r, i, st.op,
                     api.GetErrorString(nr));
  }
  return MM_OK;
}

}  // namespace
}  // namespace mmb

using namespace mmb;

extern "C" {

__attribute__((visibility("default"))) mm_status mm_window_alloc(mm_ctx* ctx, void* nccl_comm, size_t bytes, void** ptr) {
  if (!ctx || !nccl_comm || !ptr || bytes == 0)
    return ctx ? set_err(ctx, MM_ERR_USAGE, "mm_window_alloc: NULL argument or zero bytes") : MM_ERR_USAGE;
  DeviceGuard dg(ctx->device);
  const NcclApi& api = nccl_api();
  if (!api.ok) return set_err(ctx, MM_ERR_RUNTIME, "libnccl.so.2 is not loaded in this process");
  if (!api.MemAlloc || !api.MemFree || !api.CommWindowRegister || !api.CommWindowDeregister)
    return set_err(ctx, MM_ERR_UNSUPPORTED, "the loaded NCCL has no symmetric-memory window API");
  void* p = nullptr;
  NCCL_CHECK(ctx, api.MemAlloc(&p, bytes));
  ncclWindow_t w = nullptr;
  ncclResult_t rr = api.CommWindowRegister(static_cast<ncclComm_t>(nccl_comm), p, bytes, &w, NCCL_WIN_COLL_SYMMETRIC);
  if (rr != ncclSuccess) {
    api.MemFree(p);
    return set_err(ctx, MM_ERR_RUNTIME, "ncclCommWindowRegister failed: %s", api.GetErrorString(rr));
  }
  ctx->windows.push_back({p, bytes, static_cast<void*>(w), nccl_comm});
  *ptr = p;
  return MM_OK;
}

__attribute__((visibility("default"))) mm_status mm_window_free(mm_ctx* ctx, void* ptr) {
  if (!ctx || !ptr) return ctx ? set_err(ctx, MM_ERR_USAGE, "mm_window_free: NULL argument") : MM_ERR_USAGE;
  DeviceGuard dg(ctx->device);
  const NcclApi& api = nccl_api();
  for (size_t i = 0; i < ctx->windows.size(); ++i) {
    const mm_ctx::Window e = ctx->windows[i];
    if (e.base != ptr) continue;
    ctx->windows.erase(ctx->windows.begin() + (ptrdiff_t)i);
    cudaDeviceSynchronize();  // no product may still store into it
    NCCL_CHECK(ctx, api.CommWindowDeregister(static_cast<ncclComm_t>(e.comm), static_cast<ncclWindow_t>(e.win)));
    NCCL_CHECK(ctx, api.MemFree(e.base));
    return MM_OK;
  }
  return set_err(ctx, MM_ERR_USAGE, "mm_window_free: %p was not returned by mm_window_alloc on this context", ptr);
}

__attribute__((visibility("default"))) mm_status mm_ipc_export(mm_ctx* ctx, const void* dev_ptr, mm_ipc_handle* out) {
  if (!ctx || !dev_ptr || !out) return ctx ? set_err(ctx, MM_ERR_USAGE, "mm_ipc_export: NULL argument") : MM_ERR_USAGE;
  DeviceGuard dg(ctx->device);
  CUdeviceptr base = 0;
  size_t size = 0;
  GetAddrRangeFn fn = addr_range_fn();
  if (!fn || fn(&base, &size, reinterpret_cast<CUdeviceptr>(dev_ptr)) != CUDA_SUCCESS)
    return set_err(ctx, MM_ERR_USAGE, "mm_ipc_export: %p is not device memory (cuMemGetAddressRange failed)", dev_ptr);
  cudaIpcMemHandle_t h;
  if (cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)) != cudaSuccess) {
    cudaGetLastError();
    return set_err(ctx, MM_ERR_RUNTIME, "cudaIpcGetMemHandle failed for the allocation holding %p", dev_ptr);
  }
  static_assert(sizeof(cudaIpcMemHandle_t) + sizeof(uint64_t) <= sizeof(mm_ipc_handle), "mm_ipc_handle");
  memset(out, 0, sizeof *out);
  memcpy(out->bytes, &h, sizeof h);
  const uint64_t off = reinterpret_cast<uint64_t>(dev_ptr) - (uint64_t)base;
  memcpy(out->bytes + sizeof h, &off, sizeof off);
  return MM_OK;
}

__attribute__((visibility("default"))) mm_status mm_ipc_open(mm_ctx* ctx, const mm_ipc_handle* h, void** dev_ptr) {
  if (!ctx || !h || !dev_ptr) return ctx ? set_err(ctx, MM_ERR_USAGE, "mm_ipc_open: NULL argument") : MM_ERR_USAGE;
  DeviceGuard dg(ctx->device);
  cudaIpcMemHandle_t mh;
  uint64_t off = 0;
  memcpy(&mh, h->bytes, sizeof mh);
  memcpy(&off, h->bytes + sizeof mh, sizeof off);
  const std::string key(reinterpret_cast<const char*>(&mh), sizeof mh);
  void* base = nullptr;
  for (auto& mp : ctx->ipc_open)
    if (mp.handle == key) base = mp.base;
  if (!base) {
    if (cudaIpcOpenMemHandle(&base, mh, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      const cudaError_t e = cudaGetLastError();
      return set_err(ctx, MM_ERR_RUNTIME, "cudaIpcOpenMemHandle failed: %s (an allocation of this process, or no "
                     "peer access?)", cudaGetErrorString(e));
    }
    CUdeviceptr b0 = 0;
    size_t size = 0;
    GetAddrRangeFn fn = addr_range_fn();
    if (!fn || fn(&b0, &size, reinterpret_cast<CUdeviceptr>(base)) != CUDA_SUCCESS) size = 0;
    ctx->ipc_open.push_back({key, base, size});
  }
  *dev_ptr = static_cast<uint8_t*>(base) + off;
  return MM_OK;
}

void mm_release_comms(mm_ctx* ctx) {
  if (!ctx) return;
  const NcclApi& api = nccl_api();
  for (int c = 1; c < 4; ++c) {
    if (ctx->sub_comm[c] && api.CommDestroy) api.CommDestroy(static_cast<ncclComm_t>(ctx->sub_comm[c]));
    ctx->sub_comm[c] = nullptr;
  }
  for (int i = 0; i < 4; ++i) ctx->split_sig[i] = -1;
  ctx->split_parent = nullptr;
}

void mm_release_ipc(mm_ctx* ctx) {
  if (!ctx) return;
  for (auto& mp : ctx->ipc_open) cudaIpcCloseMemHandle(mp.base);
  ctx->ipc_open.clear();
  if (ctx->ipc_xchg) cudaFree(ctx->ipc_xchg);
  if (ctx->bar_buf) cudaFree(ctx->bar_buf);
  ctx->ipc_xchg = ctx->bar_buf = nullptr;
  for (cudaEvent_t e : ctx->plan_events) cudaEventDestroy(e);
  ctx->plan_events.clear();
}

__attribute__((visibility("default"))) mm_status mm_gemm_sharded(mm_ctx* ctx, int64_t m, int64_t n, int64_t p,
                                                                 mm_dtype dtype, mm_layout layout, int grid_rows,
                                                                 int grid_cols, const void* A_local, void* B_local,
                                                                 void* C_local, void* C_full, unsigned flags, int root,
                                                                 void* nccl_comm, void* stream) {
  if (!ctx) return MM_ERR_USAGE;
  knobs_refresh();
  DeviceGuard dg(ctx->device);
  if (dtype != MM_F64 && dtype != MM_BF16_F32 && dtype != MM_S8_S32 && dtype != MM_F64_EMU)
    return set_err(ctx, MM_ERR_USAGE, "unknown dtype %d", (int)dtype);
  if (m < 1 || n < 1 || p < 1) return set_err(ctx, MM_ERR_USAGE, "dimensions must be >= 1");
  if (!nccl_comm) return set_err(ctx, MM_ERR_USAGE, "nccl_comm is NULL");
  mm_status st = refuse_diag_knobs(ctx);
  if (st != MM_OK) return st;
  const NcclApi& api = nccl_api();
  if (!api.ok)
    return set_err(ctx, MM_ERR_RUNTIME, "libnccl.so.2 is not loaded in this process (set MM_NCCL_LIB to override)");
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int G = 0, r = 0;
  NCCL_CHECK(ctx, api.CommCount(comm, &G));
  NCCL_CHECK(ctx, api.CommUserRank(comm, &r));
  // Collective contract (include/mm.h): every rank passes the same (m, n, p, dtype, layout, grid,
  // flags, root).  Checked with one all-reduce of a hash and its negation (MAX of both equals the
  // hash on every rank iff all hashes agree) in the diagnostic build, or with MM_CHECK_COLLECTIVE=1
  // (it synchronises the stream, so it is off by default in the release library).
  bool check = knob("MM_CHECK_COLLECTIVE") != nullptr;
#ifdef MM_DIAG
  check = true;
#endif
  if (check) {
    uint64_t hsh = 1469598103934665603ull;
    const int64_t words[9] = {m, n, p, (int64_t)dtype, (int64_t)layout, grid_rows, grid_cols, (int64_t)flags, root};
    for (int64_t w : words) hsh = (hsh ^ (uint64_t)w) * 1099511628211ull;
    const int64_t h = (int64_t)(hsh >> 2);  // (positive)
    int64_t pair[2] = {h, -h};
    if (!ctx->bar_buf && cudaMalloc(&ctx->bar_buf, 16) != cudaSuccess)
      return set_err(ctx, MM_ERR_WORKSPACE, "barrier buffer allocation failed");
    cudaStream_t s0 = static_cast<cudaStream_t>(stream);
    if (cudaMemcpyAsync(ctx->bar_buf, pair, sizeof pair, cudaMemcpyHostToDevice, s0) != cudaSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "collective check staging failed");
    NCCL_CHECK(ctx, api.AllReduce(ctx->bar_buf, ctx->bar_buf, 2, ncclInt64, ncclMax, comm, s0));
    if (cudaMemcpyAsync(pair, ctx->bar_buf, sizeof pair, cudaMemcpyDeviceToHost, s0) != cudaSuccess ||
        cudaStreamSynchronize(s0) != cudaSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "collective check failed");
    if (pair[0] != h || pair[1] != -h)
      return set_err(ctx, MM_ERR_USAGE, "rank %d: mm_gemm_sharded arguments differ across the %d ranks "
                     "(m, n, p, dtype, layout, grid, flags and root must match)", r, G);
  }
  // argument errors with messages (mm_shard_plan applies the same rules)
  if (layout == MM_ROW_BLOCK) {
    if (root < 0 || root >= G) return set_err(ctx, MM_ERR_USAGE, "root %d outside [0, %d)", root, G);
    if (!B_local) return set_err(ctx, MM_ERR_USAGE, "B_local is NULL");
    if ((flags & MM_GATHER_C) && (flags & MM_GATHER_C_FUSED))
      return set_err(ctx, MM_ERR_USAGE, "MM_GATHER_C and MM_GATHER_C_FUSED are exclusive");
    if (flags & ~(unsigned)(MM_BCAST_B | MM_GATHER_C | MM_GATHER_C_FUSED | MM_C_WINDOW))
      return set_err(ctx, MM_ERR_USAGE, "MM_ROW_BLOCK takes MM_BCAST_B | MM_GATHER_C | MM_GATHER_C_FUSED | MM_C_WINDOW only");
    if ((flags & MM_C_WINDOW) && !(flags & MM_GATHER_C_FUSED))
      return set_err(ctx, MM_ERR_USAGE, "MM_C_WINDOW applies to MM_GATHER_C_FUSED only");
    if ((flags & MM_C_WINDOW) && !C_full)
      return set_err(ctx, MM_ERR_USAGE, "MM_C_WINDOW: every rank passes its own window buffer as C_full (NULL on rank %d)", r);
    if ((flags & (MM_GATHER_C | MM_GATHER_C_FUSED)) && r == root && !C_full)
      return set_err(ctx, MM_ERR_USAGE, "MM_GATHER_C / MM_GATHER_C_FUSED need C_full on the root rank");
  } else if (layout == MM_SUMMA_2D || layout == MM_SUMMA_25D) {
    if (dtype != MM_F64 && dtype != MM_F64_EMU)
      return set_err(ctx, MM_ERR_UNSUPPORTED, "MM_SUMMA_2D/25D accumulate across k-panels; implemented for MM_F64 and MM_F64_EMU");
    if (layout == MM_SUMMA_2D && (grid_rows < 1 || grid_cols < 1 || grid_rows * grid_cols != G))
      return set_err(ctx, MM_ERR_USAGE, "grid %d x %d does not match communicator size %d", grid_rows, grid_cols, G);
    if (layout == MM_SUMMA_2D && flags)
      return set_err(ctx, MM_ERR_USAGE, "MM_SUMMA_2D takes no flags (operands and C stay block-distributed)");
    if (layout == MM_SUMMA_25D && (grid_rows < 1 || grid_cols < 1 || G % (grid_rows * grid_cols) != 0))
      return set_err(ctx, MM_ERR_USAGE, "grid %d x %d does not divide communicator size %d", grid_rows, grid_cols, G);
    if (layout == MM_SUMMA_25D && (flags & ~(unsigned)MM_REPLICATE))
      return set_err(ctx, MM_ERR_USAGE, "MM_SUMMA_25D takes only MM_REPLICATE");
  } else {
    return set_err(ctx, MM_ERR_USAGE, "unknown layout %d", (int)layout);
  }
  mm_plan_info info;
  st = mm_shard_plan(m, n, p, dtype, layout, grid_rows, grid_cols, flags, root, G, r, 0, nullptr, 0, &info);
  if (st != MM_OK) return set_err(ctx, st, "mm_shard_plan rejected the arguments (rank %d of %d)", r, G);
  std::vector<mm_plan_step> steps((size_t)info.steps);
  mm_shard_plan(m, n, p, dtype, layout, grid_rows, grid_cols, flags, root, G, r, 0, steps.data(), info.steps, &info);
  PlanBufs B;
  B.p[MM_BUF_A] = static_cast<uint8_t*>(const_cast<void*>(A_local));
  B.p[MM_BUF_B] = static_cast<uint8_t*>(B_local);
  B.p[MM_BUF_C] = static_cast<uint8_t*>(C_local);
  B.p[MM_BUF_CFULL] = static_cast<uint8_t*>(C_full);
  B.c_window = layout == MM_ROW_BLOCK && (flags & MM_C_WINDOW);
  // the sub-communicator cache key: identical on every rank (ROW_BLOCK splits nothing)
  const int64_t sig[4] = {(int64_t)layout, layout == MM_ROW_BLOCK ? 0 : grid_rows, layout == MM_ROW_BLOCK ? 0 : grid_cols,
                          (int64_t)G};
  return execute_plan(ctx, steps, info, B, dtype, comm, r, sig, static_cast<cudaStream_t>(stream));
}

}  // extern "C"
