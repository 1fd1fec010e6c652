"""paper_2408_15384_b200 — B200-native (sm_100a) dense product C = A·B.

The paper's hot path (§III): C[i][j] = Σ_k A[i][k]·B[k][j]
for an m×n A and an n×p B, row-major.  The compute runs in
libmm_b200.so (tcgen05 for BF16/INT8, DMMA for FP64, TMA-fed); this module
marshals torch tensors into the C-ABI of include/mm.h.  PyTorch supplies only
device memory, streams and process groups.

    import paper_2408_15384_b200 as mm
    C = mm.gemm(A, B)            # A, B on cuda: float64 | bfloat16 | int8
    C = mm.gemm_host(A, B)       # A, B on the host (pinned for full PCIe rate)
"""
from __future__ import annotations

import ctypes
import threading

import torch

from . import _lib
from ._lib import (MM_BCAST_B, MM_BF16_F32, MM_C_WINDOW, MM_F64, MM_F64_EMU, MM_GATHER_C, MM_GATHER_C_FUSED,
                   MM_REPLICATE, MM_ROW_BLOCK, MM_S8_S32, MM_SUMMA_2D, MM_SUMMA_25D)

__all__ = ["gemm", "gemm_host", "gemm_sharded", "shard_range", "summa_panels", "shard_plan", "workspace_size",
           "ipc_export", "ipc_open", "window_alloc", "window_free", "clock_meter", "MMError", "Context",
           "sync_check", "version", "launches", "MM_F64", "MM_BF16_F32", "MM_S8_S32", "MM_ROW_BLOCK", "MM_SUMMA_2D",
           "MM_BCAST_B", "MM_GATHER_C", "MM_GATHER_C_FUSED", "MM_REPLICATE", "MM_SUMMA_25D",
           "MM_C_WINDOW", "MM_F64_EMU"]

IN_DTYPE = {torch.float64: MM_F64, torch.bfloat16: MM_BF16_F32, torch.int8: MM_S8_S32}
OUT_DTYPE = {MM_F64: torch.float64, MM_BF16_F32: torch.float32, MM_S8_S32: torch.int32, MM_F64_EMU: torch.float64}


class MMError(RuntimeError):
    def __init__(self, status: int, msg: str):
        self.status = status
        super().__init__(f"{_lib.load().mm_status_string(status).decode()}: {msg}")


class Context:
    """Owns one mm_ctx (per device, per thread)."""

    def __init__(self, device: int = 0, workspace: torch.Tensor | None = None):
        lib = _lib.load()
        h = ctypes.c_void_p()
        ws_ptr = workspace.data_ptr() if workspace is not None else None
        ws_bytes = workspace.numel() * workspace.element_size() if workspace is not None else 0
        st = lib.mm_create(device, ws_ptr, ws_bytes, ctypes.byref(h))
        if st != 0:
            raise MMError(st, f"mm_create(device={device}) failed")
        self.handle = h
        self.device = device
        self._ws = workspace

    def check(self, st: int):
        if st != 0:
            raise MMError(st, _lib.load().mm_last_error(self.handle).decode())

    def close(self):
        if self.handle:
            _lib.load().mm_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_local = threading.local()
_MM_GEMM = None  # mm_gemm, resolved on first use


def context(device: int | None = None) -> Context:
    if device is None:
        device = torch.cuda.current_device()
    cache = getattr(_local, "ctx", None)
    if cache is None:
        cache = _local.ctx = {}
    if device not in cache:
        cache[device] = Context(device)
    return cache[device]


def launches(device: int | None = None) -> int:
    """Kernels launched so far by this thread's context on `device`."""
    return int(_lib.load().mm_launches(context(device).handle))


def version() -> str:
    return _lib.load().mm_version().decode()


def _check_operands(A: torch.Tensor, B: torch.Tensor):
    if A.dim() != 2 or B.dim() != 2:
        raise ValueError(f"A and B must be 2-D, got {tuple(A.shape)} and {tuple(B.shape)}")
    if A.shape[1] != B.shape[0]:
        raise ValueError(f"inner dimensions differ: A is {tuple(A.shape)}, B is {tuple(B.shape)}")
    if A.dtype != B.dtype or A.dtype not in IN_DTYPE:
        raise TypeError(f"A and B must share a dtype in {list(IN_DTYPE)}; got {A.dtype}, {B.dtype}")
    if not (A.is_contiguous() and B.is_contiguous()):
        raise ValueError("A and B must be contiguous row-major")
    return A.shape[0], A.shape[1], B.shape[1], IN_DTYPE[A.dtype]


try:  # the raw current-stream handle without constructing a torch.cuda.Stream (~2 us per call)
    _raw_stream = torch._C._cuda_getCurrentRawStream
except AttributeError:  # pragma: no cover
    def _raw_stream(idx):
        return torch.cuda.current_stream(idx).cuda_stream


def gemm(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None,
         stream: torch.cuda.Stream | None = None, f64_emulation: bool = False) -> torch.Tensor:
    """C = A·B on the GPU (async on `stream`, default: torch's current stream).
    f64_emulation (float64 operands): MM_F64_EMU, the binary64 product on the INT8 tensor cores."""
    m, n, p, dt = _check_operands(A, B)
    if f64_emulation:
        if dt != MM_F64:
            raise ValueError("f64_emulation needs float64 operands")
        dt = MM_F64_EMU
    dev = A.device
    if dev.type != "cuda" or B.device != dev:
        raise ValueError("gemm expects A and B on the same CUDA device (use gemm_host for host operands)")
    if out is None:
        out = torch.empty((m, p), dtype=OUT_DTYPE[dt], device=dev)
    elif out.shape != (m, p) or out.dtype != OUT_DTYPE[dt] or not out.is_contiguous() or out.device != dev:
        raise ValueError(f"out must be a contiguous {OUT_DTYPE[dt]} ({m}, {p}) tensor on {dev}")
    idx = dev.index if dev.index is not None else torch.cuda.current_device()
    ctx = context(idx)
    sh = stream.cuda_stream if stream is not None else _raw_stream(idx)
    global _MM_GEMM
    if _MM_GEMM is None:
        _MM_GEMM = _lib.load().mm_gemm
    st = _MM_GEMM(ctx.handle, m, n, p, dt, A.data_ptr(), B.data_ptr(), out.data_ptr(), sh)
    if st:
        ctx.check(st)
    return out


def gemm_host(A: torch.Tensor, B: torch.Tensor, out: torch.Tensor | None = None, device: int = 0,
              f64_emulation: bool = False) -> torch.Tensor:
    """C = A·B with host operands (copies in, computes, copies out; synchronous);
    f64_emulation (float64 operands): each block as MM_F64_EMU."""
    m, n, p, dt = _check_operands(A, B)
    if f64_emulation:
        dt = _dtype_code(A.dtype, True)
    if A.is_cuda or B.is_cuda:
        raise ValueError("gemm_host expects host tensors")
    if out is None:
        out = torch.empty((m, p), dtype=OUT_DTYPE[dt], pin_memory=A.is_pinned())
    ctx = context(device)
    with torch.cuda.device(device):
        s = torch.cuda.current_stream(device)
        ctx.check(_lib.load().mm_gemm_host(ctx.handle, m, n, p, dt, A.data_ptr(), B.data_ptr(), out.data_ptr(),
                                           s.cuda_stream))
    return out


def sync_check(device: int | None = None, stream: torch.cuda.Stream | None = None):
    """Synchronize and raise if a kernel latched a pipeline error."""
    ctx = context(device)
    s = stream if stream is not None else torch.cuda.current_stream(ctx.device)
    ctx.check(_lib.load().mm_sync_check(ctx.handle, s.cuda_stream))


def shard_range(total: int, G: int, r: int) -> tuple[int, int]:
    """(start, count) of part r of `total` split over G parts (⌈total/G⌉ rule)."""
    s, c = ctypes.c_int64(), ctypes.c_int64()
    _lib.load().mm_shard_range(total, G, r, ctypes.byref(s), ctypes.byref(c))
    return s.value, c.value


def summa_panels(n: int, grid_rows: int, grid_cols: int, panel: int):
    """SUMMA k-panel schedule: list of (k0, kw, a_col_owner, b_row_owner)."""
    lib = _lib.load()
    cnt = lib.mm_summa_panels(n, grid_rows, grid_cols, panel, 0, None, None, None, None)
    k0 = (ctypes.c_int64 * cnt)()
    kw = (ctypes.c_int64 * cnt)()
    ao = (ctypes.c_int * cnt)()
    bo = (ctypes.c_int * cnt)()
    lib.mm_summa_panels(n, grid_rows, grid_cols, panel, cnt, k0, kw, ao, bo)
    return [(k0[i], kw[i], ao[i], bo[i]) for i in range(cnt)]


def _dtype_code(dtype: torch.dtype, f64_emulation: bool) -> int:
    if f64_emulation:
        if dtype != torch.float64:
            raise ValueError("f64_emulation needs float64 operands")
        return MM_F64_EMU
    return IN_DTYPE[dtype]


def shard_plan(m: int, n: int, p: int, dtype: torch.dtype, *, layout: int = MM_ROW_BLOCK,
               grid: tuple[int, int] = (0, 0), flags: int = 0, root: int = 0, world: int = 1, rank: int = 0,
               panel: int = 0, f64_emulation: bool = False):
    """The plan rank `rank` of `world` runs for mm_gemm_sharded (include/mm.h, mm_shard_plan):
    (steps, info) with steps a list of dicts (op/buffer/communicator names resolved) and info a dict
    with the communicator split colours/keys and the staging-buffer sizes."""
    lib = _lib.load()
    info = _lib.PlanInfo()
    dt = _dtype_code(dtype, f64_emulation)
    st = lib.mm_shard_plan(m, n, p, dt, layout, grid[0], grid[1], flags, root, world, rank, panel, None, 0,
                           ctypes.byref(info))
    if st != 0:
        raise MMError(st, f"mm_shard_plan(m={m}, n={n}, p={p}, layout={layout}, grid={grid}, flags={flags}, "
                          f"root={root}, world={world}, rank={rank}) rejected the arguments")
    arr = (_lib.PlanStep * max(1, info.steps))()
    lib.mm_shard_plan(m, n, p, dt, layout, grid[0], grid[1], flags, root, world, rank, panel, arr, info.steps,
                      ctypes.byref(info))
    steps = []
    for i in range(info.steps):
        s = arr[i]
        d = {f: getattr(s, f) for f, _ in _lib.PlanStep._fields_}
        d["op"] = _lib.OPS[s.op]
        for b in ("dst", "src", "src2"):
            d[b] = _lib.BUFS[getattr(s, b)]
        d["comm"] = _lib.COMMS[s.comm]
        steps.append(d)
    meta = {"events": info.events, "color": {_lib.COMMS[c]: info.color[c] for c in range(4)},
            "key": {_lib.COMMS[c]: info.key[c] for c in range(4)}, "stage_bytes": list(info.stage_bytes)}
    return steps, meta


def workspace_size(m: int, n: int, p: int, dtype: torch.dtype, layout: int = MM_ROW_BLOCK, world: int = 1,
                   f64_emulation: bool = False) -> int:
    """Upper bound of the device scratch a context allocates for such a call (mm_workspace_size)."""
    return int(_lib.load().mm_workspace_size(m, n, p, _dtype_code(dtype, f64_emulation), layout, world))


def ipc_export(t: torch.Tensor) -> bytes:
    """CUDA-IPC handle (72 bytes) of the device memory at t.data_ptr() (mm_ipc_export)."""
    ctx = context(t.device.index)
    h = _lib.IpcHandle()
    ctx.check(_lib.load().mm_ipc_export(ctx.handle, t.data_ptr(), ctypes.byref(h)))
    return bytes(h.bytes)


def ipc_open(handle: bytes, device: int = 0) -> int:
    """Map another process's exported device memory (mm_ipc_open); returns the device address."""
    ctx = context(device)
    h = _lib.IpcHandle()
    ctypes.memmove(h.bytes, handle, 72)
    ptr = ctypes.c_void_p()
    ctx.check(_lib.load().mm_ipc_open(ctx.handle, ctypes.byref(h), ctypes.byref(ptr)))
    return int(ptr.value)


class _DevBuf:
    """A raw device buffer seen through __cuda_array_interface__ (torch.as_tensor wraps it, no copy)."""

    def __init__(self, ptr: int, shape, typestr: str):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": typestr, "data": (ptr, False),
                                         "version": 3, "strides": None, "stream": None}


_TYPESTR = {torch.float64: "<f8", torch.float32: "<f4", torch.int32: "<i4", torch.bfloat16: "<i2", torch.int8: "|i1"}


def window_alloc(shape, dtype: torch.dtype, group=None, device: int | None = None) -> torch.Tensor:
    """Collective (mm_window_alloc): NCCL symmetric memory for MM_GATHER_C_FUSED | MM_C_WINDOW,
    returned as a tensor viewing this rank's buffer.  Free it with window_free (collective)."""
    dev = torch.cuda.current_device() if device is None else device
    ctx = context(dev)
    numel = 1
    for d in shape:
        numel *= int(d)
    nbytes = numel * torch.empty(0, dtype=dtype).element_size()
    ptr = ctypes.c_void_p()
    ctx.check(_lib.load().mm_window_alloc(ctx.handle, _nccl_comm_ptr(group), nbytes, ctypes.byref(ptr)))
    t = torch.as_tensor(_DevBuf(int(ptr.value), shape, _TYPESTR[dtype]), device=torch.device("cuda", dev))
    return t.view(dtype) if dtype == torch.bfloat16 else t


def window_free(t: torch.Tensor):
    """Collective (mm_window_free): deregister and free a window_alloc buffer."""
    ctx = context(t.device.index)
    ctx.check(_lib.load().mm_window_free(ctx.handle, t.data_ptr()))


def gemm_ptr(m: int, n: int, p: int, dtype: torch.dtype, A: int, B: int, C: int, device: int = 0,
             stream: torch.cuda.Stream | None = None):
    """C = A·B on raw device addresses (e.g. C mapped with ipc_open); async on `stream`."""
    ctx = context(device)
    sh = stream.cuda_stream if stream is not None else _raw_stream(device)
    ctx.check(_lib.load().mm_gemm(ctx.handle, m, n, p, IN_DTYPE[dtype], A, B, C, sh))


def clock_meter(enable: bool, device: int | None = None) -> float:
    """mm_clock_meter: start recording (returns 0.0), or stop and return the effective SM clock
    (MHz) of the most recent product kernel of this thread's context on `device`."""
    ctx = context(device)
    mhz = ctypes.c_double()
    ctx.check(_lib.load().mm_clock_meter(ctx.handle, 1 if enable else 0, ctypes.byref(mhz)))
    return float(mhz.value)


def _nccl_comm_ptr(group) -> int:
    import torch.distributed as dist
    pg = group if group is not None else dist.group.WORLD
    backend = pg._get_backend(torch.device("cuda", torch.cuda.current_device()))
    return backend._comm_ptr()


def gemm_sharded(m: int, n: int, p: int, dtype: torch.dtype, A_local: torch.Tensor | None,
                 B_local: torch.Tensor, C_local: torch.Tensor | None, *, layout: int = MM_ROW_BLOCK,
                 grid: tuple[int, int] = (0, 0), flags: int = 0, root: int = 0,
                 C_full: torch.Tensor | None = None, group=None, stream: torch.cuda.Stream | None = None,
                 f64_emulation: bool = False):
    """Collective product over an NCCL process group (see include/mm.h, mm_gemm_sharded);
    f64_emulation (float64): every local product as MM_F64_EMU."""
    dt = _dtype_code(dtype, f64_emulation)
    dev = B_local.device
    ctx = context(dev.index)
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    comm = _nccl_comm_ptr(group)

    def ptr(t):
        return t.data_ptr() if t is not None and t.numel() > 0 else None
    ctx.check(_lib.load().mm_gemm_sharded(ctx.handle, m, n, p, dt, layout, grid[0], grid[1], ptr(A_local),
                                          ptr(B_local), ptr(C_local), ptr(C_full), flags, root, comm,
                                          s.cuda_stream))
