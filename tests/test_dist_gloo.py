"""Multi-process host logic of the sharded layouts, world_size 2 on CPU (gloo).

Each rank runs the same schedule the library's mm_gemm_sharded runs (shard
ranges from mm_shard_range, k-panels from mm_summa_panels, broadcast roots,
gather order), with torch.distributed/gloo standing in for NCCL and the CPU
oracle standing in for the local GPU product.  The assembled C must equal the
single-process oracle product bit for bit (exact-integer inputs), i.e. the
partition and exchange logic is exact (SPEC.md:210 G-invariance)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as tmp

import oracle
import paper_2408_15384_b200 as mm
import synthgen as sg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _inputs(m, n, p):
    return sg.exact_f64(21, 1, 2049, m, n), sg.exact_f64(21, 2, 2049, n, p)


def _row_block_worker(rank, world, port, m, n, p, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B = _inputs(m, n, p)
        root = world - 1
        s, c = mm.shard_range(m, world, rank)
        A_local = torch.from_numpy(A[s:s + c].copy())
        # MM_BCAST_B: only the root has B
        B_local = torch.from_numpy(B.copy()) if rank == root else torch.zeros(n, p, dtype=torch.float64)
        dist.broadcast(B_local, src=root)
        C_local = torch.from_numpy(oracle.gemm_f64(A_local.numpy(), B_local.numpy())) if c else torch.zeros(0, p, dtype=torch.float64)
        # MM_GATHER_C: ragged shards -> send/recv to root in rank order
        if rank == root:
            C_full = torch.zeros(m, p, dtype=torch.float64)
            for r in range(world):
                rs, rc = mm.shard_range(m, world, r)
                if rc == 0:
                    continue
                if r == rank:
                    C_full[rs:rs + rc] = C_local
                else:
                    buf = torch.zeros(rc, p, dtype=torch.float64)
                    dist.recv(buf, src=r)
                    C_full[rs:rs + rc] = buf
            q.put(("C", C_full.numpy()))
        elif c:
            dist.send(C_local, dst=root)
    finally:
        dist.destroy_process_group()


def _summa_worker(rank, world, port, m, n, p, pr, pc, panel, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        A, B = _inputs(m, n, p)
        gi, gj = rank // pc, rank % pc
        am, ak = mm.shard_range(m, pr, gi), mm.shard_range(n, pc, gj)
        bk, bn = mm.shard_range(n, pr, gi), mm.shard_range(p, pc, gj)
        A_loc = A[am[0]:am[0] + am[1], ak[0]:ak[0] + ak[1]]
        B_loc = B[bk[0]:bk[0] + bk[1], bn[0]:bn[0] + bn[1]]
        row_groups = [dist.new_group([i * pc + j for j in range(pc)]) for i in range(pr)]
        col_groups = [dist.new_group([i * pc + j for i in range(pr)]) for j in range(pc)]
        C_loc = np.zeros((am[1], bn[1]))
        for (k0, kw, ao, bo) in mm.summa_panels(n, pr, pc, panel):
            Ap = torch.zeros(am[1], kw, dtype=torch.float64)
            if gj == ao:
                Ap[:] = torch.from_numpy(np.ascontiguousarray(A_loc[:, k0 - ak[0]:k0 - ak[0] + kw]))
            dist.broadcast(Ap, src=gi * pc + ao, group=row_groups[gi])
            Bp = torch.zeros(kw, bn[1], dtype=torch.float64)
            if gi == bo:
                Bp[:] = torch.from_numpy(np.ascontiguousarray(B_loc[k0 - bk[0]:k0 - bk[0] + kw]))
            dist.broadcast(Bp, src=bo * pc + gj, group=col_groups[gj])
            if am[1] and bn[1]:
                C_loc += oracle.gemm_f64(Ap.numpy(), Bp.numpy())  # beta=1 accumulate over panels
        q.put(("blk", rank, C_loc))
    finally:
        dist.destroy_process_group()


def _summa25_worker(rank, world, port, m, n, p, pr, pc, panel, q):
    """MM_SUMMA_25D schedule: layer l = rank // (pr*pc) runs the SUMMA panels t ≡ l (mod c)
    on its copy of the blocks (MM_REPLICATE: broadcast from layer 0 along the depth), then
    the layers' C blocks are summed onto layer 0."""
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        c = world // (pr * pc)
        A, B = _inputs(m, n, p)
        l, r2 = rank // (pr * pc), rank % (pr * pc)
        gi, gj = r2 // pc, r2 % pc
        am, ak = mm.shard_range(m, pr, gi), mm.shard_range(n, pc, gj)
        bk, bn = mm.shard_range(n, pr, gi), mm.shard_range(p, pc, gj)
        rank_of = lambda ll, i, j: ll * pr * pc + i * pc + j  # noqa: E731
        row_groups = {(ll, i): dist.new_group([rank_of(ll, i, j) for j in range(pc)]) for ll in range(c) for i in range(pr)}
        col_groups = {(ll, j): dist.new_group([rank_of(ll, i, j) for i in range(pr)]) for ll in range(c) for j in range(pc)}
        depth_groups = {(i, j): dist.new_group([rank_of(ll, i, j) for ll in range(c)]) for i in range(pr) for j in range(pc)}
        # MM_REPLICATE: only layer 0 holds the blocks
        A_loc = torch.zeros(am[1], ak[1], dtype=torch.float64)
        B_loc = torch.zeros(bk[1], bn[1], dtype=torch.float64)
        if l == 0:
            A_loc[:] = torch.from_numpy(np.ascontiguousarray(A[am[0]:am[0] + am[1], ak[0]:ak[0] + ak[1]]))
            B_loc[:] = torch.from_numpy(np.ascontiguousarray(B[bk[0]:bk[0] + bk[1], bn[0]:bn[0] + bn[1]]))
        dist.broadcast(A_loc, src=rank_of(0, gi, gj), group=depth_groups[(gi, gj)])
        dist.broadcast(B_loc, src=rank_of(0, gi, gj), group=depth_groups[(gi, gj)])
        A_loc, B_loc = A_loc.numpy(), B_loc.numpy()
        C_loc = torch.zeros(am[1], bn[1], dtype=torch.float64)
        panels = mm.summa_panels(n, pr, pc, panel)
        for t in range(l, len(panels), c):
            k0, kw, ao, bo = panels[t]
            Ap = torch.zeros(am[1], kw, dtype=torch.float64)
            if gj == ao:
                Ap[:] = torch.from_numpy(np.ascontiguousarray(A_loc[:, k0 - ak[0]:k0 - ak[0] + kw]))
            dist.broadcast(Ap, src=rank_of(l, gi, ao), group=row_groups[(l, gi)])
            Bp = torch.zeros(kw, bn[1], dtype=torch.float64)
            if gi == bo:
                Bp[:] = torch.from_numpy(np.ascontiguousarray(B_loc[k0 - bk[0]:k0 - bk[0] + kw]))
            dist.broadcast(Bp, src=rank_of(l, bo, gj), group=col_groups[(l, gj)])
            C_loc += torch.from_numpy(oracle.gemm_f64(Ap.numpy(), Bp.numpy()))
        dist.reduce(C_loc, dst=rank_of(0, gi, gj), op=dist.ReduceOp.SUM, group=depth_groups[(gi, gj)])
        if l == 0:
            q.put(("blk", rank, C_loc.numpy()))
    finally:
        dist.destroy_process_group()


def _spawn(target, args, world):
    ctx = tmp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=target, args=(r, world, port) + args + (q,)) for r in range(world)]
    for pr_ in procs:
        pr_.start()
    out = []
    for pr_ in procs:
        pr_.join(timeout=180)
        assert pr_.exitcode == 0, f"worker exit code {pr_.exitcode}"
    while not q.empty():
        out.append(q.get())
    return out


@pytest.mark.parametrize("m,n,p", [(37, 19, 23), (2, 5, 3), (1, 4, 4), (64, 48, 80)])
def test_row_block_world2_equals_single_process(m, n, p):
    out = _spawn(_row_block_worker, (m, n, p), 2)
    (_, C), = [o for o in out if o[0] == "C"]
    A, B = _inputs(m, n, p)
    assert np.array_equal(C, oracle.gemm_f64(A, B))


@pytest.mark.parametrize("pr,pc", [(1, 2), (2, 1)])
@pytest.mark.parametrize("m,n,p,panel", [(37, 41, 29, 8), (16, 16, 16, 16), (5, 3, 7, 1)])
def test_summa_world2_equals_single_process(pr, pc, m, n, p, panel):
    out = _spawn(_summa_worker, (m, n, p, pr, pc, panel), 2)
    A, B = _inputs(m, n, p)
    C = oracle.gemm_f64(A, B)
    blocks = {o[1]: o[2] for o in out if o[0] == "blk"}
    assert len(blocks) == 2
    for rank, blk in blocks.items():
        gi, gj = rank // pc, rank % pc
        am, bn = mm.shard_range(m, pr, gi), mm.shard_range(p, pc, gj)
        # exact-integer entries: every summation order gives the same bits
        assert np.array_equal(blk, C[am[0]:am[0] + am[1], bn[0]:bn[0] + bn[1]])


@pytest.mark.parametrize("world,pr,pc", [(2, 1, 1), (4, 2, 1), (4, 1, 2)])
@pytest.mark.parametrize("m,n,p,panel", [(37, 41, 29, 8), (9, 3, 11, 1)])
def test_summa25d_equals_single_process(world, pr, pc, m, n, p, panel):
    out = _spawn(_summa25_worker, (m, n, p, pr, pc, panel), world)
    A, B = _inputs(m, n, p)
    C = oracle.gemm_f64(A, B)
    blocks = {o[1]: o[2] for o in out if o[0] == "blk"}
    assert len(blocks) == pr * pc  # layer 0 holds the result
    for rank, blk in blocks.items():
        gi, gj = rank // pc, rank % pc
        am, bn = mm.shard_range(m, pr, gi), mm.shard_range(p, pc, gj)
        assert np.array_equal(blk, C[am[0]:am[0] + am[1], bn[0]:bn[0] + bn[1]])
