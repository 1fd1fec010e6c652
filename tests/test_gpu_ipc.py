"""The non-root half of MM_GATHER_C_FUSED on one GPU: two processes, a CUDA-IPC mapping, TMA stores.

In a fused row-block gather every non-root rank maps the root's C_full (mm_ipc_open of the handle
mm_ipc_export made on the root) and its product kernel stores its C tiles through that mapping.
NCCL refuses two ranks on one GPU, so here the two halves run as two processes on the same
device, the 72-byte handle travelling over gloo — the same library calls (mm_ipc_export,
mm_ipc_open, a product whose C lies in the mapping: plain TMA stores, no reduce-add tail) that
rank r > 0 makes in the fused path (csrc/shard.cu peer_pointer_of_root).  The root then checks the
whole C_full against the oracle bit for bit (exact-integer inputs)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu

CASES = [("bf16", 1000, 2560, 2560), ("i8", 777, 4096, 1300), ("f64", 900, 1500, 1750), ("bf16", 4096, 512, 4096)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(dt, m, n, p):
    if dt == "bf16":
        return sg.exact_bf16(95, 1, 9, m, n), sg.exact_bf16(95, 2, 9, n, p)
    if dt == "i8":
        return sg.exact_i8(95, 1, 255, m, n), sg.exact_i8(95, 2, 255, n, p)
    return sg.exact_f64(95, 1, 2049, m, n), sg.exact_f64(95, 2, 2049, n, p)


def _dev(x, dt):
    if dt == "bf16":
        return torch.from_numpy(np.ascontiguousarray(x).view(np.int16)).view(torch.bfloat16).cuda()
    return torch.from_numpy(np.ascontiguousarray(x)).cuda()


def _worker(rank, port, q):
    import paper_2408_15384_b200 as mm
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=2)
    torch.cuda.set_device(0)
    try:
        for (dt, m, n, p) in CASES:
            A, B = _inputs(dt, m, n, p)
            tdt = {"bf16": torch.bfloat16, "i8": torch.int8, "f64": torch.float64}[dt]
            odt = {"bf16": torch.float32, "i8": torch.int32, "f64": torch.float64}[dt]
            s, c = mm.shard_range(m, 2, rank)
            Ad, Bd = _dev(A[s:s + c], dt), _dev(B, dt)
            eo = torch.empty(0, dtype=odt).element_size()
            if rank == 0:
                big = torch.full((m + 5, p), -3, dtype=odt, device="cuda")
                C_full = big[2:2 + m]  # inside a larger allocation: the handle carries the offset
                obj = [mm.ipc_export(C_full)]
            else:
                obj = [None]
            dist.broadcast_object_list(obj, src=0)
            if rank == 0:
                mm.gemm(Ad, Bd, out=C_full[s:s + c])
            else:
                base = mm.ipc_open(obj[0])
                mm.gemm_ptr(c, n, p, tdt, Ad.data_ptr(), Bd.data_ptr(), base + s * p * eo)
            mm.sync_check()
            torch.cuda.synchronize()
            dist.barrier()
            if rank == 0:
                Cref = {"bf16": lambda: oracle.gemm_bf16(A, B)[0], "i8": lambda: oracle.gemm_s8(A, B),
                        "f64": lambda: oracle.gemm_f64(A, B)}[dt]()
                h = big.cpu().numpy().astype(np.float64)
                ok = np.array_equal(h[2:2 + m], np.asarray(Cref, np.float64))
                guards = bool(np.all(h[:2] == -3) and np.all(h[2 + m:] == -3))
                q.put((dt, m, n, p, ok, guards))
            dist.barrier()  # the root's allocation outlives the peer's use of the mapping
    finally:
        dist.destroy_process_group()


def test_fused_gather_non_root_half_one_gpu(cuda_device):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, port, q)) for r in range(2)]
    for pr in procs:
        pr.start()
    try:
        res = [q.get(timeout=600) for _ in CASES]
    finally:
        for pr in procs:
            pr.join(timeout=120)
    assert all(pr.exitcode == 0 for pr in procs), [pr.exitcode for pr in procs]
    for (dt, m, n, p, ok, guards) in res:
        assert ok, (dt, m, n, p)
        assert guards, (dt, m, n, p)
