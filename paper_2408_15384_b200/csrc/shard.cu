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
  bool ok = false;
};
NcclApi g_nccl;
std::once_flag g_nccl_once;

const NcclApi& nccl() {
  std::call_once(g_nccl_once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOLOAD | RTLD_LAZY);
    if (!h) {
      const char* p = getenv("MM_NCCL_LIB");
      if (p) h = dlopen(p, RTLD_LAZY | RTLD_GLOBAL);
    }
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
      return set_err(ctx, MM_ERR_RUNTIME, "%s failed: %s", #call, nccl().GetErrorString(_r));               \
  } while (0)

struct Range {
  int64_t start, count;
};

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

// Collective: every rank learns a pointer to the root's `root_ptr` it can store to
// (the root's own pointer on the root; a CUDA-IPC mapping of the root's allocation,
// over NVLink, elsewhere).  The 64-byte IPC handle + offset travel by ncclBroadcast.
mm_status peer_pointer_of_root(mm_ctx* ctx, void* root_ptr, int root, int r, ncclComm_t comm, cudaStream_t s,
                               uint8_t** out) {
  struct Msg {
    cudaIpcMemHandle_t h;
    uint64_t offset;
  } msg;
  memset(&msg, 0, sizeof msg);
  if (r == root) {
    CUdeviceptr base = 0;
    size_t size = 0;
    GetAddrRangeFn fn = addr_range_fn();
    if (!fn || fn(&base, &size, reinterpret_cast<CUdeviceptr>(root_ptr)) != CUDA_SUCCESS)
      return set_err(ctx, MM_ERR_RUNTIME, "cuMemGetAddressRange failed for C_full");
    if (cudaIpcGetMemHandle(&msg.h, reinterpret_cast<void*>(base)) != cudaSuccess) {
      cudaGetLastError();
      return set_err(ctx, MM_ERR_RUNTIME, "cudaIpcGetMemHandle failed for C_full");
    }
    msg.offset = reinterpret_cast<uint64_t>(root_ptr) - (uint64_t)base;
  }
  if (!ctx->ipc_xchg && cudaMalloc(&ctx->ipc_xchg, 256) != cudaSuccess)
    return set_err(ctx, MM_ERR_WORKSPACE, "IPC exchange buffer allocation failed");
  if (r == root && cudaMemcpyAsync(ctx->ipc_xchg, &msg, sizeof msg, cudaMemcpyHostToDevice, s) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "IPC handle staging failed");
  NCCL_CHECK(ctx, nccl().Broadcast(ctx->ipc_xchg, ctx->ipc_xchg, sizeof msg, ncclUint8, root, comm, s));
  if (cudaMemcpyAsync(&msg, ctx->ipc_xchg, sizeof msg, cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "IPC handle exchange failed");
  if (r == root) {
    *out = static_cast<uint8_t*>(root_ptr);
    return MM_OK;
  }
  const std::string key(reinterpret_cast<const char*>(&msg.h), sizeof msg.h);
  void* base = nullptr;
  for (auto& kv : ctx->ipc_open)
    if (kv.first == key) base = kv.second;
  if (!base) {
    if (cudaIpcOpenMemHandle(&base, msg.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      return set_err(ctx, MM_ERR_RUNTIME, "cudaIpcOpenMemHandle of the root's C_full failed (peer access?)");
    }
    ctx->ipc_open.emplace_back(key, base);
  }
  *out = static_cast<uint8_t*>(base) + msg.offset;
  return MM_OK;
}
Range shard(int64_t total, int G, int r) {
  Range x;
  mm_shard_range(total, G, r, &x.start, &x.count);
  return x;
}

}  // namespace
}  // namespace mmb

using namespace mmb;

extern "C" {

__attribute__((visibility("default"))) void mm_shard_range(int64_t total, int G, int r, int64_t* start,
                                                           int64_t* count) {
  int64_t s = 0, c = 0;
  if (G >= 1 && r >= 0 && r < G && total > 0) {
    const int64_t q = (total + G - 1) / G;  // ⌈total/G⌉
    s = std::min<int64_t>((int64_t)r * q, total);
    c = std::min<int64_t>(q, total - s);
  }
  if (start) *start = s;
  if (count) *count = c;
}

__attribute__((visibility("default"))) int mm_summa_panels(int64_t n, int grid_rows, int grid_cols, int64_t panel,
                                                           int cap, int64_t* k0, int64_t* kw, int* a_col,
                                                           int* b_row) {
  if (n < 1 || grid_rows < 1 || grid_cols < 1 || panel < 1) return 0;
  // boundaries = union of A's column-block and B's row-block boundaries along k
  std::vector<int64_t> cuts = {0, n};
  for (int j = 0; j < grid_cols; ++j) cuts.push_back(shard(n, grid_cols, j).start);
  for (int i = 0; i < grid_rows; ++i) cuts.push_back(shard(n, grid_rows, i).start);
  std::sort(cuts.begin(), cuts.end());
  cuts.erase(std::unique(cuts.begin(), cuts.end()), cuts.end());
  int np = 0;
  for (size_t c = 0; c + 1 < cuts.size(); ++c) {
    for (int64_t k = cuts[c]; k < cuts[c + 1]; k += panel) {
      const int64_t w = std::min<int64_t>(panel, cuts[c + 1] - k);
      if (np < cap) {
        if (k0) k0[np] = k;
        if (kw) kw[np] = w;
        int oa = 0, ob = 0;
        for (int j = 0; j < grid_cols; ++j) {
          Range r = shard(n, grid_cols, j);
          if (k >= r.start && k < r.start + r.count) oa = j;
        }
        for (int i = 0; i < grid_rows; ++i) {
          Range r = shard(n, grid_rows, i);
          if (k >= r.start && k < r.start + r.count) ob = i;
        }
        if (a_col) a_col[np] = oa;
        if (b_row) b_row[np] = ob;
      }
      ++np;
    }
  }
  return np;
}

void mm_release_comms(mm_ctx* ctx) {
  if (!ctx) return;
  for (auto& kv : ctx->ipc_open) cudaIpcCloseMemHandle(kv.second);
  ctx->ipc_open.clear();
  if (ctx->ipc_xchg) cudaFree(ctx->ipc_xchg);
  if (ctx->bar_buf) cudaFree(ctx->bar_buf);
  ctx->ipc_xchg = ctx->bar_buf = nullptr;
  const NcclApi& api = nccl();
  if (api.CommDestroy) {
    if (ctx->row_comm) api.CommDestroy(static_cast<ncclComm_t>(ctx->row_comm));
    if (ctx->col_comm) api.CommDestroy(static_cast<ncclComm_t>(ctx->col_comm));
    if (ctx->depth_comm) api.CommDestroy(static_cast<ncclComm_t>(ctx->depth_comm));
  }
  ctx->row_comm = ctx->col_comm = ctx->depth_comm = nullptr;
  ctx->split_parent = nullptr;
}

static mm_status row_block(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, const void* A_local,
                           void* B_local, void* C_local, void* C_full, unsigned flags, int root, ncclComm_t comm,
                           int G, int r, cudaStream_t s) {
  const NcclApi& api = nccl();
  const size_t ei = dtype_in_size(dtype), eo = dtype_out_size(dtype);
  const Range mine = shard(m, G, r);

  // Where this rank's C rows go: its own C_local, or (MM_GATHER_C_FUSED) straight into the
  // root's C_full over NVLink — GEMM -> gather as ONE kernel per rank (TMA stores to peer memory).
  uint8_t* target = static_cast<uint8_t*>(C_local);
  if (flags & MM_GATHER_C_FUSED) {
    if (r == root && !C_full) return set_err(ctx, MM_ERR_USAGE, "MM_GATHER_C_FUSED needs C_full on the root rank");
    uint8_t* full = nullptr;
    mm_status st = peer_pointer_of_root(ctx, C_full, root, r, comm, s, &full);
    if (st != MM_OK) return st;
    target = full + mine.start * p * eo;
  }
  // products into a peer's memory: plain TMA stores only (no reduce-add split tail over NVLink)
  struct RemoteC {
    mm_ctx* c;
    RemoteC(mm_ctx* c_, bool on) : c(c_) { c->c_remote = on ? 1 : 0; }
    ~RemoteC() { c->c_remote = 0; }
  } remote_c(ctx, (flags & MM_GATHER_C_FUSED) != 0);

  if (flags & MM_BCAST_B) {
    // B broadcast in column panels, double-buffered on a communication stream, so the
    // broadcast of panel j+1 overlaps the product C[:, panel j] = A · B[:, panel j].
    int64_t npan = 8;
    if (const char* e = knob("MM_BCAST_PANELS")) npan = std::max<int64_t>(1, atoll(e));  // tuning knob
    int64_t w = (p + npan - 1) / npan;
    w = (w + 15) / 16 * 16;  // 16-element multiple: every panel pitch is 16-B aligned for TMA
    if (w > p) w = p;
    const int64_t J = (p + w - 1) / w;
    mm_status st;
    for (int b = 0; b < 2; ++b)
      if ((st = ensure_buffer(ctx, &ctx->sbuf[b], &ctx->sbuf_bytes[b], (size_t)(n * w) * ei)) != MM_OK) return st;
    if (!ctx->s_in && cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking) != cudaSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "stream creation failed");
    cudaStream_t sc = ctx->s_in;
    cudaEvent_t ev_start, ev_ready[2], ev_free[2], ev_end;
    cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_end, cudaEventDisableTiming);
    for (int b = 0; b < 2; ++b) {
      cudaEventCreateWithFlags(&ev_ready[b], cudaEventDisableTiming);
      cudaEventCreateWithFlags(&ev_free[b], cudaEventDisableTiming);
    }
    cudaEventRecord(ev_start, s);
    cudaStreamWaitEvent(sc, ev_start, 0);
    st = MM_OK;
    for (int64_t j = 0; j < J && st == MM_OK; ++j) {
      const int b = (int)(j & 1);
      const int64_t c0 = j * w, wj = std::min(w, p - c0);
      uint8_t* stage = static_cast<uint8_t*>(ctx->sbuf[b]);
      uint8_t* Bcol = static_cast<uint8_t*>(B_local) + c0 * ei;
      if (j >= 2) cudaStreamWaitEvent(sc, ev_free[b], 0);
      if (r == root && cudaMemcpy2DAsync(stage, (size_t)wj * ei, Bcol, (size_t)p * ei, (size_t)wj * ei, (size_t)n,
                                         cudaMemcpyDeviceToDevice, sc) != cudaSuccess) {
        st = set_err(ctx, MM_ERR_RUNTIME, "B panel staging failed");
        break;
      }
      ncclResult_t nr = api.Broadcast(stage, stage, (size_t)(n * wj) * ei, ncclUint8, root, comm, sc);
      if (nr != ncclSuccess) {
        st = set_err(ctx, MM_ERR_RUNTIME, "B panel broadcast failed: %s", api.GetErrorString(nr));
        break;
      }
      // keep the contract "B_local holds B afterwards" on every rank (off the critical path)
      if (r != root && cudaMemcpy2DAsync(Bcol, (size_t)p * ei, stage, (size_t)wj * ei, (size_t)wj * ei, (size_t)n,
                                         cudaMemcpyDeviceToDevice, sc) != cudaSuccess) {
        st = set_err(ctx, MM_ERR_RUNTIME, "B panel copy-out failed");
        break;
      }
      cudaEventRecord(ev_ready[b], sc);
      cudaStreamWaitEvent(s, ev_ready[b], 0);
      if (mine.count > 0)
        st = gemm_ld(ctx, mine.count, n, wj, dtype, A_local, n, stage, wj, target + c0 * eo, p, 0, s);
      cudaEventRecord(ev_free[b], s);
    }
    cudaEventRecord(ev_end, sc);
    cudaStreamWaitEvent(s, ev_end, 0);
    cudaEventDestroy(ev_start);
    cudaEventDestroy(ev_end);
    for (int b = 0; b < 2; ++b) {
      cudaEventDestroy(ev_ready[b]);
      cudaEventDestroy(ev_free[b]);
    }
    if (st != MM_OK) return st;
  } else if (mine.count > 0) {
    mm_status st = gemm_ld(ctx, mine.count, n, p, dtype, A_local, n, B_local, p, target, p, 0, s);
    if (st != MM_OK) return st;
  }

  if (flags & MM_GATHER_C_FUSED) {
    // barrier: the root's C_full is complete once every rank's product kernels have finished
    if (!ctx->bar_buf && cudaMalloc(&ctx->bar_buf, 16) != cudaSuccess)
      return set_err(ctx, MM_ERR_WORKSPACE, "barrier buffer allocation failed");
    NCCL_CHECK(ctx, api.AllReduce(ctx->bar_buf, ctx->bar_buf, 1, ncclInt32, ncclSum, comm, s));
    return MM_OK;
  }
  if (flags & MM_GATHER_C) {
    if (r == root && !C_full) return set_err(ctx, MM_ERR_USAGE, "MM_GATHER_C needs C_full on the root rank");
    NCCL_CHECK(ctx, api.GroupStart());
    if (r == root) {
      for (int q = 0; q < G; ++q) {
        const Range rq = shard(m, G, q);
        if (rq.count == 0) continue;
        uint8_t* dst = static_cast<uint8_t*>(C_full) + rq.start * p * eo;
        if (q == r) {
          if (cudaMemcpyAsync(dst, C_local, (size_t)(rq.count * p) * eo, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
            return set_err(ctx, MM_ERR_RUNTIME, "local copy into C_full failed");
        } else {
          NCCL_CHECK(ctx, api.Recv(dst, (size_t)(rq.count * p) * eo, ncclUint8, q, comm, s));
        }
      }
    } else if (mine.count > 0) {
      NCCL_CHECK(ctx, api.Send(C_local, (size_t)(mine.count * p) * eo, ncclUint8, root, comm, s));
    }
    NCCL_CHECK(ctx, api.GroupEnd());
  }
  return MM_OK;
}

// SUMMA over a pr × pc grid, replicated over `layers` depth layers (2.5D, Solomonik &
// Demmel; "2.5D Matrix Multiplication").  Rank r ↔ (layer l, gi, gj) with
// r = l·pr·pc + gi·pc + gj.  Every layer holds the same A/B blocks; layer l runs the SUMMA
// k-panels t ≡ l (mod layers), so each layer broadcasts 1/layers of the panels, and the
// layers' partial C blocks are summed onto layer 0 by an NCCL reduce along the depth
// communicator.  layers = 1 is plain SUMMA.
static mm_status summa_2d(mm_ctx* ctx, int64_t m, int64_t n, int64_t p, mm_dtype dtype, int pr, int pc,
                          int layers, const void* A_local, const void* B_local, void* C_local, ncclComm_t comm,
                          int r, unsigned flags, cudaStream_t s) {
  const NcclApi& api = nccl();
  if (dtype != MM_F64)
    return set_err(ctx, MM_ERR_UNSUPPORTED, "MM_SUMMA_2D/25D accumulate across k-panels; implemented for MM_F64");
  const size_t ei = dtype_in_size(dtype);
  const int l = r / (pr * pc), r2 = r % (pr * pc);
  const int gi = r2 / pc, gj = r2 % pc;
  // sub-communicators: grid row (color l·pr+gi, rank gj), grid column (color l·pc+gj, rank gi),
  // depth (color gi·pc+gj, rank l)
  if (ctx->split_parent != comm || ctx->split_rows != pr || ctx->split_cols != pc || ctx->split_layers != layers) {
    mm_release_comms(ctx);
    ncclComm_t rc = nullptr, cc = nullptr, dc = nullptr;
    NCCL_CHECK(ctx, api.CommSplit(comm, l * pr + gi, gj, &rc, nullptr));
    NCCL_CHECK(ctx, api.CommSplit(comm, l * pc + gj, gi, &cc, nullptr));
    if (layers > 1) NCCL_CHECK(ctx, api.CommSplit(comm, gi * pc + gj, l, &dc, nullptr));
    ctx->row_comm = rc;
    ctx->col_comm = cc;
    ctx->depth_comm = dc;
    ctx->split_parent = comm;
    ctx->split_rows = pr;
    ctx->split_cols = pc;
    ctx->split_layers = layers;
  }
  ncclComm_t row_comm = static_cast<ncclComm_t>(ctx->row_comm);
  ncclComm_t col_comm = static_cast<ncclComm_t>(ctx->col_comm);
  ncclComm_t depth_comm = static_cast<ncclComm_t>(ctx->depth_comm);

  const Range am = shard(m, pr, gi), ak = shard(n, pc, gj);  // my A block: rows am, cols ak
  const Range bk = shard(n, pr, gi), bn = shard(p, pc, gj);  // my B block: rows bk, cols bn
  if (layers > 1 && (flags & MM_REPLICATE)) {
    // the caller placed the blocks on layer 0 only: replicate them along the depth
    NCCL_CHECK(ctx, api.GroupStart());
    if (am.count > 0 && ak.count > 0)
      NCCL_CHECK(ctx, api.Broadcast(A_local, const_cast<void*>(A_local), (size_t)(am.count * ak.count) * ei, ncclUint8,
                                    0, depth_comm, s));
    if (bk.count > 0 && bn.count > 0)
      NCCL_CHECK(ctx, api.Broadcast(B_local, const_cast<void*>(B_local), (size_t)(bk.count * bn.count) * ei, ncclUint8,
                                    0, depth_comm, s));
    NCCL_CHECK(ctx, api.GroupEnd());
  }
  int64_t panel = 2048;
  if (const char* e = knob("MM_SUMMA_PANEL")) panel = std::max<int64_t>(16, atoll(e));
  const int np = mm_summa_panels(n, pr, pc, panel, 0, nullptr, nullptr, nullptr, nullptr);
  std::vector<int64_t> k0(np), kw(np);
  std::vector<int> ao(np), bo(np);
  mm_summa_panels(n, pr, pc, panel, np, k0.data(), kw.data(), ao.data(), bo.data());

  // two buffer sets {A panel (am.count × panel), B panel (panel × bn.count)}
  const size_t abytes = (size_t)(std::max<int64_t>(am.count, 1) * panel) * ei;
  const size_t bbytes = (size_t)(panel * std::max<int64_t>(bn.count, 1)) * ei;
  mm_status st;
  for (int b = 0; b < 2; ++b) {
    if ((st = ensure_buffer(ctx, &ctx->sbuf[2 * b], &ctx->sbuf_bytes[2 * b], abytes)) != MM_OK) return st;
    if ((st = ensure_buffer(ctx, &ctx->sbuf[2 * b + 1], &ctx->sbuf_bytes[2 * b + 1], bbytes)) != MM_OK) return st;
  }
  if (!ctx->s_in && cudaStreamCreateWithFlags(&ctx->s_in, cudaStreamNonBlocking) != cudaSuccess)
    return set_err(ctx, MM_ERR_RUNTIME, "stream creation failed");
  cudaStream_t sc = ctx->s_in;  // communication stream
  cudaEvent_t ev_ready[2], ev_free[2], ev_start;
  for (int b = 0; b < 2; ++b) {
    cudaEventCreateWithFlags(&ev_ready[b], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&ev_free[b], cudaEventDisableTiming);
  }
  cudaEventCreateWithFlags(&ev_start, cudaEventDisableTiming);
  cudaEventRecord(ev_start, s);
  cudaStreamWaitEvent(sc, ev_start, 0);
  // C block starts at zero if some panel never reaches us (empty k range cannot happen: n >= 1)
  st = MM_OK;
  int done = 0;  // panels this layer has accumulated
  for (int t = l; t < np && st == MM_OK; t += layers) {
    const int b = (t / layers) & 1;
    uint8_t* Ap = static_cast<uint8_t*>(ctx->sbuf[2 * b]);
    uint8_t* Bp = static_cast<uint8_t*>(ctx->sbuf[2 * b + 1]);
    if (done >= 2) cudaStreamWaitEvent(sc, ev_free[b], 0);
    // owners stage their panel into the send buffer (A: a column slice → pitched copy; B: whole rows)
    if (gj == ao[t] && am.count > 0) {
      const uint8_t* src = static_cast<const uint8_t*>(A_local) + (size_t)(k0[t] - ak.start) * ei;
      if (cudaMemcpy2DAsync(Ap, (size_t)kw[t] * ei, src, (size_t)ak.count * ei, (size_t)kw[t] * ei, (size_t)am.count,
                            cudaMemcpyDeviceToDevice, sc) != cudaSuccess) {
        st = set_err(ctx, MM_ERR_RUNTIME, "A panel copy failed");
        break;
      }
    }
    if (gi == bo[t] && bn.count > 0) {
      const uint8_t* src = static_cast<const uint8_t*>(B_local) + (size_t)((k0[t] - bk.start) * bn.count) * ei;
      if (cudaMemcpyAsync(Bp, src, (size_t)(kw[t] * bn.count) * ei, cudaMemcpyDeviceToDevice, sc) != cudaSuccess) {
        st = set_err(ctx, MM_ERR_RUNTIME, "B panel copy failed");
        break;
      }
    }
    ncclResult_t nr = api.GroupStart();
    if (nr == ncclSuccess && am.count > 0)
      nr = api.Broadcast(Ap, Ap, (size_t)(am.count * kw[t]) * ei, ncclUint8, ao[t], row_comm, sc);
    if (nr == ncclSuccess && bn.count > 0)
      nr = api.Broadcast(Bp, Bp, (size_t)(kw[t] * bn.count) * ei, ncclUint8, bo[t], col_comm, sc);
    ncclResult_t ne = api.GroupEnd();
    if (nr != ncclSuccess || ne != ncclSuccess) {
      st = set_err(ctx, MM_ERR_RUNTIME, "SUMMA panel broadcast failed: %s",
                   api.GetErrorString(nr != ncclSuccess ? nr : ne));
      break;
    }
    cudaEventRecord(ev_ready[b], sc);
    cudaStreamWaitEvent(s, ev_ready[b], 0);
    if (am.count > 0 && bn.count > 0)
      st = gemm_ld(ctx, am.count, kw[t], bn.count, dtype, Ap, kw[t], Bp, bn.count, C_local, bn.count, done > 0 ? 1 : 0,
                   s);
    cudaEventRecord(ev_free[b], s);
    ++done;
  }
  // the caller's stream must not run ahead of the last communication
  cudaEvent_t ev_end;
  cudaEventCreateWithFlags(&ev_end, cudaEventDisableTiming);
  cudaEventRecord(ev_end, sc);
  cudaStreamWaitEvent(s, ev_end, 0);
  cudaEventDestroy(ev_end);
  for (int b = 0; b < 2; ++b) {
    cudaEventDestroy(ev_ready[b]);
    cudaEventDestroy(ev_free[b]);
  }
  cudaEventDestroy(ev_start);
  if (st != MM_OK) return st;
  if (layers > 1 && am.count > 0 && bn.count > 0) {
    // a layer that received no panel contributes zeros; then sum the layers onto layer 0
    if (done == 0 && cudaMemsetAsync(C_local, 0, (size_t)(am.count * bn.count) * ei, s) != cudaSuccess)
      return set_err(ctx, MM_ERR_RUNTIME, "zeroing C_local failed");
    NCCL_CHECK(ctx, api.Reduce(C_local, C_local, (size_t)(am.count * bn.count), ncclFloat64, ncclSum, 0, depth_comm, s));
  }
  return MM_OK;
}

__attribute__((visibility("default"))) mm_status mm_gemm_sharded(mm_ctx* ctx, int64_t m, int64_t n, int64_t p,
                                                                 mm_dtype dtype, mm_layout layout, int grid_rows,
                                                                 int grid_cols, const void* A_local, void* B_local,
                                                                 void* C_local, void* C_full, unsigned flags, int root,
                                                                 void* nccl_comm, void* stream) {
  if (!ctx) return MM_ERR_USAGE;
  knobs_refresh();
  DeviceGuard dg(ctx->device);
  if (!ctx) return MM_ERR_USAGE;
  if (dtype != MM_F64 && dtype != MM_BF16_F32 && dtype != MM_S8_S32)
    return set_err(ctx, MM_ERR_USAGE, "unknown dtype %d", (int)dtype);
  if (m < 1 || n < 1 || p < 1) return set_err(ctx, MM_ERR_USAGE, "dimensions must be >= 1");
  if (!nccl_comm) return set_err(ctx, MM_ERR_USAGE, "nccl_comm is NULL");
  const NcclApi& api = nccl();
  if (!api.ok)
    return set_err(ctx, MM_ERR_RUNTIME, "libnccl.so.2 is not loaded in this process (set MM_NCCL_LIB to override)");
  ncclComm_t comm = static_cast<ncclComm_t>(nccl_comm);
  int G = 0, r = 0;
  NCCL_CHECK(ctx, api.CommCount(comm, &G));
  NCCL_CHECK(ctx, api.CommUserRank(comm, &r));
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (layout == MM_ROW_BLOCK) {
    if (root < 0 || root >= G) return set_err(ctx, MM_ERR_USAGE, "root %d outside [0, %d)", root, G);
    if (!B_local) return set_err(ctx, MM_ERR_USAGE, "B_local is NULL");
    const Range mine = shard(m, G, r);
    if (mine.count > 0 && (!A_local || (!C_local && !(flags & MM_GATHER_C_FUSED))))
      return set_err(ctx, MM_ERR_USAGE, "NULL A_local/C_local");
    return row_block(ctx, m, n, p, dtype, A_local, B_local, C_local, C_full, flags, root, comm, G, r, s);
  }
  if (layout == MM_SUMMA_2D) {
    if (grid_rows < 1 || grid_cols < 1 || grid_rows * grid_cols != G)
      return set_err(ctx, MM_ERR_USAGE, "grid %d x %d does not match communicator size %d", grid_rows, grid_cols, G);
    if (flags) return set_err(ctx, MM_ERR_USAGE, "MM_SUMMA_2D takes no flags (operands and C stay block-distributed)");
    return summa_2d(ctx, m, n, p, dtype, grid_rows, grid_cols, 1, A_local, B_local, C_local, comm, r, 0, s);
  }
  if (layout == MM_SUMMA_25D) {
    if (grid_rows < 1 || grid_cols < 1 || G % (grid_rows * grid_cols) != 0)
      return set_err(ctx, MM_ERR_USAGE, "grid %d x %d does not divide communicator size %d", grid_rows, grid_cols, G);
    if (flags & ~(unsigned)MM_REPLICATE) return set_err(ctx, MM_ERR_USAGE, "MM_SUMMA_25D takes only MM_REPLICATE");
    return summa_2d(ctx, m, n, p, dtype, grid_rows, grid_cols, G / (grid_rows * grid_cols), A_local, B_local, C_local,
                    comm, r, flags, s);
  }
  return set_err(ctx, MM_ERR_USAGE, "unknown layout %d", (int)layout);
}

}  // extern "C"
