// fake_nccl.cu — TEST ONLY.  A stand-in for the handful of NCCL entry points the library resolves
// (csrc/shard.cu), for several processes sharing ONE GPU — which real NCCL refuses ("duplicate
// GPU").  It lets tests/test_gpu_shim_multirank.py run the library's real sharded executor and
// product kernels at world sizes 2-4 on a one-GPU box, for correctness only:
//   * every call first synchronises its stream, then does blocking work on the host: buffers are
//     exchanged through CUDA IPC (cudaIpcGetMemHandle / OpenMemHandle) and cudaMemcpy, ranks meet at
//     process-shared barriers in a POSIX shared-memory segment;
//   * no kernel ever waits for another rank, and nothing here is timed.
// Loaded by the library through MM_NCCL_LIB; the test obtains a world communicator from
// fake_comm_init(rank, nranks, shm_name).
#include <cuda.h>
#include <cuda_runtime.h>
#include <fcntl.h>
#include <nccl.h>
#include <sched.h>
#include <sys/mman.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstdlib>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <vector>

namespace {

constexpr int kMaxRanks = 8;
constexpr int kMaxComms = 256;  // comm id = split sequence * 8 + (colour & 7)

struct Barrier {
  std::atomic<uint32_t> count;
  std::atomic<uint32_t> gen;
};
struct Slot {
  cudaIpcMemHandle_t h;
  uint64_t off, bytes;
};
struct Mailbox {  // src -> dst point-to-point channel
  std::atomic<uint32_t> posted, acked;
  Slot slot;
};
struct Shared {
  Barrier world_bar;
  Barrier comm_bar[kMaxComms];
  Slot slots[kMaxComms][kMaxRanks];
  int split_color[kMaxComms][kMaxRanks], split_key[kMaxComms][kMaxRanks];
  Mailbox mbox[kMaxRanks][kMaxRanks];
};

struct Comm {
  int id;                         // shared-state index
  std::vector<int> members;       // world ranks, in comm-rank order
  int rank;                       // this process's rank in the comm
};

Shared* g_sh = nullptr;
int g_world_rank = -1, g_world_n = 0;
int g_split_seq = 0;
int g_group = 0;
struct Pending {
  int kind;  // 0 send, 1 recv, 2 broadcast, 3 allreduce, 4 reduce
  const void* sbuf;
  void* rbuf;
  size_t bytes, count;
  ncclDataType_t dt;
  ncclRedOp_t op;
  int peer;
  Comm* comm;
};
std::vector<Pending> g_pending;

void barrier(Barrier& b, int n) {
  const uint32_t g = b.gen.load();
  if (b.count.fetch_add(1) + 1 == (uint32_t)n) {
    b.count.store(0);
    b.gen.fetch_add(1);
  } else {
    while (b.gen.load() == g) sched_yield();
  }
}
void comm_barrier(Comm* c) { barrier(g_sh->comm_bar[c->id], (int)c->members.size()); }

size_t dt_size(ncclDataType_t t) {
  switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    case ncclInt64: case ncclUint64: case ncclFloat64: return 8;
    default: return 2;
  }
}

// export a device buffer (any pointer inside an allocation)
bool export_buf(const void* p, size_t bytes, Slot* s) {
  CUdeviceptr base = 0;
  size_t size = 0;
  if (cuMemGetAddressRange(&base, &size, (CUdeviceptr)p) != CUDA_SUCCESS) return false;
  if (cudaIpcGetMemHandle(&s->h, (void*)base) != cudaSuccess) return false;
  s->off = (uint64_t)((CUdeviceptr)p - base);
  s->bytes = bytes;
  return true;
}
// copy `bytes` from a peer's exported buffer into `dst` (device) or to host when dst_host
bool fetch(const Slot& s, void* dst, size_t bytes, bool to_host) {
  void* base = nullptr;
  if (cudaIpcOpenMemHandle(&base, s.h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) return false;
  const cudaError_t e = cudaMemcpy(dst, (char*)base + s.off, bytes, to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
  cudaIpcCloseMemHandle(base);
  return e == cudaSuccess;
}

template <typename T>
void combine(std::vector<char>& acc, const std::vector<char>& x, size_t count, ncclRedOp_t op) {
  T* a = reinterpret_cast<T*>(acc.data());
  const T* b = reinterpret_cast<const T*>(x.data());
  for (size_t i = 0; i < count; ++i) a[i] = op == ncclMax ? (a[i] > b[i] ? a[i] : b[i]) : a[i] + b[i];
}
void combine_any(std::vector<char>& acc, const std::vector<char>& x, size_t count, ncclDataType_t dt, ncclRedOp_t op) {
  if (dt == ncclFloat64) combine<double>(acc, x, count, op);
  else if (dt == ncclInt64) combine<int64_t>(acc, x, count, op);
  else if (dt == ncclFloat32) combine<float>(acc, x, count, op);
  else combine<int32_t>(acc, x, count, op);
}

ncclResult_t do_broadcast(const void* sbuf, void* rbuf, size_t bytes, int root, Comm* c) {
  if (c->rank == root) {
    if (sbuf != rbuf && cudaMemcpy(rbuf, sbuf, bytes, cudaMemcpyDeviceToDevice) != cudaSuccess) return ncclUnhandledCudaError;
    if (!export_buf(rbuf, bytes, &g_sh->slots[c->id][root])) return ncclUnhandledCudaError;
  }
  comm_barrier(c);
  bool ok = true;
  if (c->rank != root) ok = fetch(g_sh->slots[c->id][root], rbuf, bytes, false);
  comm_barrier(c);
  return ok ? ncclSuccess : ncclUnhandledCudaError;
}

// all-reduce (reduce when root >= 0: only the root's recvbuff is written)
ncclResult_t do_reduce(const void* sbuf, void* rbuf, size_t count, ncclDataType_t dt, ncclRedOp_t op, int root, Comm* c) {
  const size_t bytes = count * dt_size(dt);
  if (!export_buf(sbuf, bytes, &g_sh->slots[c->id][c->rank])) return ncclUnhandledCudaError;
  comm_barrier(c);
  bool ok = true;
  if (root < 0 || c->rank == root) {
    std::vector<char> acc(bytes), x(bytes);
    for (int q = 0; q < (int)c->members.size() && ok; ++q) {  // member order: fixed
      char* dst = q == 0 ? acc.data() : x.data();
      if (q == c->rank)  // (an allocation of this process cannot be IPC-opened here)
        ok = cudaMemcpy(dst, sbuf, bytes, cudaMemcpyDeviceToHost) == cudaSuccess;
      else
        ok = fetch(g_sh->slots[c->id][q], dst, bytes, true);
      if (ok && q > 0) combine_any(acc, x, count, dt, op);
    }
    comm_barrier(c);  // every rank has read every send buffer before any is overwritten
    if (ok) ok = cudaMemcpy(rbuf, acc.data(), bytes, cudaMemcpyHostToDevice) == cudaSuccess;
  } else {
    comm_barrier(c);
  }
  comm_barrier(c);
  return ok ? ncclSuccess : ncclUnhandledCudaError;
}

ncclResult_t run(const Pending& p) {
  switch (p.kind) {
    case 2: return do_broadcast(p.sbuf, p.rbuf, p.bytes, p.peer, p.comm);
    case 3: return do_reduce(p.sbuf, p.rbuf, p.count, p.dt, p.op, -1, p.comm);
    case 4: return do_reduce(p.sbuf, p.rbuf, p.count, p.dt, p.op, p.peer, p.comm);
    default: return ncclInternalError;
  }
}

// point-to-point inside GroupEnd: post every send, serve every receive, then wait for the acks
ncclResult_t flush_p2p(std::vector<Pending>& ops) {
  for (auto& p : ops)
    if (p.kind == 0) {
      const int dst = p.comm->members[p.peer];
      Mailbox& mb = g_sh->mbox[g_world_rank][dst];
      while (mb.posted.load() != mb.acked.load()) sched_yield();  // previous message consumed
      if (!export_buf(p.sbuf, p.bytes, &mb.slot)) return ncclUnhandledCudaError;
      mb.posted.fetch_add(1);
    }
  for (auto& p : ops)
    if (p.kind == 1) {
      const int src = p.comm->members[p.peer];
      Mailbox& mb = g_sh->mbox[src][g_world_rank];
      while (mb.posted.load() == mb.acked.load()) sched_yield();
      const bool ok = mb.slot.bytes == p.bytes && fetch(mb.slot, p.rbuf, p.bytes, false);
      mb.acked.fetch_add(1);
      if (!ok) return ncclUnhandledCudaError;
    }
  for (auto& p : ops)
    if (p.kind == 0) {
      Mailbox& mb = g_sh->mbox[g_world_rank][p.comm->members[p.peer]];
      while (mb.posted.load() != mb.acked.load()) sched_yield();
    }
  return ncclSuccess;
}

bool g_debug = getenv("FAKE_NCCL_DEBUG") != nullptr;

ncclResult_t submit(Pending p, cudaStream_t s) {
  if (g_debug)
    fprintf(stderr, "[fake %d] op %d comm %d (rank %d of %zu) bytes %zu peer %d group %d\n", g_world_rank, p.kind,
            p.comm->id, p.comm->rank, p.comm->members.size(), p.bytes, p.peer, g_group);
  if (cudaStreamSynchronize(s) != cudaSuccess) return ncclUnhandledCudaError;
  if (g_group > 0) {
    g_pending.push_back(p);
    return ncclSuccess;
  }
  if (p.kind <= 1) {
    std::vector<Pending> one{p};
    return flush_p2p(one);
  }
  return run(p);
}

}  // namespace

extern "C" {

// Test entry: map (creating if needed) the shared segment and return this rank's world communicator.
void* fake_comm_init(int rank, int nranks, const char* shm_name) {
  if (nranks > kMaxRanks) return nullptr;
  const int fd = shm_open(shm_name, O_CREAT | O_RDWR, 0600);
  if (fd < 0) return nullptr;
  if (ftruncate(fd, sizeof(Shared)) != 0) return nullptr;
  void* p = mmap(nullptr, sizeof(Shared), PROT_READ | PROT_WRITE, MAP_SHARED, fd, 0);
  close(fd);
  if (p == MAP_FAILED) return nullptr;
  g_sh = static_cast<Shared*>(p);  // zero-filled by ftruncate on creation
  g_world_rank = rank;
  g_world_n = nranks;
  cudaFree(nullptr);  // context
  Comm* c = new Comm{0, {}, rank};
  for (int q = 0; q < nranks; ++q) c->members.push_back(q);
  barrier(g_sh->world_bar, nranks);
  return c;
}

ncclResult_t ncclBroadcast(const void* s, void* r, size_t count, ncclDataType_t dt, int root, ncclComm_t comm,
                           cudaStream_t st) {
  return submit(Pending{2, s, r, count * dt_size(dt), count, dt, ncclSum, root, reinterpret_cast<Comm*>(comm)}, st);
}
ncclResult_t ncclAllReduce(const void* s, void* r, size_t count, ncclDataType_t dt, ncclRedOp_t op, ncclComm_t comm,
                           cudaStream_t st) {
  return submit(Pending{3, s, r, count * dt_size(dt), count, dt, op, -1, reinterpret_cast<Comm*>(comm)}, st);
}
ncclResult_t ncclReduce(const void* s, void* r, size_t count, ncclDataType_t dt, ncclRedOp_t op, int root,
                        ncclComm_t comm, cudaStream_t st) {
  return submit(Pending{4, s, r, count * dt_size(dt), count, dt, op, root, reinterpret_cast<Comm*>(comm)}, st);
}
ncclResult_t ncclSend(const void* s, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
  return submit(Pending{0, s, nullptr, count * dt_size(dt), count, dt, ncclSum, peer, reinterpret_cast<Comm*>(comm)}, st);
}
ncclResult_t ncclRecv(void* r, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t st) {
  return submit(Pending{1, nullptr, r, count * dt_size(dt), count, dt, ncclSum, peer, reinterpret_cast<Comm*>(comm)}, st);
}
ncclResult_t ncclGroupStart() {
  ++g_group;
  return ncclSuccess;
}
ncclResult_t ncclGroupEnd() {
  if (--g_group > 0) return ncclSuccess;
  std::vector<Pending> ops;
  ops.swap(g_pending);
  std::vector<Pending> p2p;
  for (auto& p : ops)
    if (p.kind <= 1) p2p.push_back(p);
  ncclResult_t r = p2p.empty() ? ncclSuccess : flush_p2p(p2p);
  for (auto& p : ops)
    if (r == ncclSuccess && p.kind >= 2) r = run(p);  // collectives in program order (same on every rank)
  return r;
}
ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t* newcomm, ncclConfig_t*) {
  Comm* parent = reinterpret_cast<Comm*>(comm);
  if (parent->id != 0) return ncclInvalidUsage;  // splits of WORLD only (what the library does)
  const int seq = ++g_split_seq;
  if (seq >= kMaxComms / 8) return ncclInternalError;
  g_sh->split_color[seq][g_world_rank] = color;
  g_sh->split_key[seq][g_world_rank] = key;
  barrier(g_sh->world_bar, g_world_n);
  Comm* c = new Comm{seq * 8 + (color & 7), {}, 0};
  std::vector<std::pair<int, int>> mem;  // (key, world rank)
  for (int q = 0; q < g_world_n; ++q)
    if (g_sh->split_color[seq][q] == color) mem.push_back({g_sh->split_key[seq][q], q});
  std::sort(mem.begin(), mem.end());
  for (size_t i = 0; i < mem.size(); ++i) {
    c->members.push_back(mem[i].second);
    if (mem[i].second == g_world_rank) c->rank = (int)i;
  }
  barrier(g_sh->world_bar, g_world_n);
  if (g_debug) fprintf(stderr, "[fake %d] split seq %d color %d key %d -> id %d rank %d of %zu\n", g_world_rank, seq,
                       color, key, c->id, c->rank, c->members.size());
  *newcomm = reinterpret_cast<ncclComm_t>(c);
  return ncclSuccess;
}
ncclResult_t ncclCommDestroy(ncclComm_t) { return ncclSuccess; }
ncclResult_t ncclCommCount(const ncclComm_t comm, int* count) {
  *count = (int)reinterpret_cast<const Comm*>(comm)->members.size();
  return ncclSuccess;
}
ncclResult_t ncclCommUserRank(const ncclComm_t comm, int* rank) {
  *rank = reinterpret_cast<const Comm*>(comm)->rank;
  return ncclSuccess;
}
const char* ncclGetErrorString(ncclResult_t r) { return r == ncclSuccess ? "fake: success" : "fake: failure"; }

}  // extern "C"
