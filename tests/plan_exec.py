"""A second executor of the library's sharded plans (include/mm.h, mm_shard_plan), for CPU tests.

The library computes, per rank, the list of steps mm_gemm_sharded runs (local products, pitched
copies, NCCL collectives, stream events).  This module runs the SAME list with torch.distributed
over gloo standing in for NCCL and the CPU oracle standing in for the local GPU product, steps in
plan order (a valid sequential order of the two streams).  Whatever the plan gets wrong — a shard
offset, a pitch, a broadcast root, a missing panel, the gather order — shows up as a wrong C.

`check_stream_order` is a static check of the plan's events: it replays the two streams with vector
clocks and asserts that every pair of conflicting buffer accesses on different streams is ordered
by a record/wait edge, and that the caller's stream ends after all communication.

Test infrastructure: may call oracle/.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.distributed as dist

import oracle

IN_NP = {"f64": np.float64, "bf16": np.uint16, "i8": np.int8}
OUT_NP = {"f64": np.float64, "bf16": np.float32, "i8": np.int32}


def _view(buf: np.ndarray, off: int, rows: int, cols: int, ld: int, dt) -> np.ndarray:
    isz = np.dtype(dt).itemsize
    if rows == 0 or cols == 0:
        return np.zeros((rows, cols), dt)
    assert off % isz == 0 and off + ((rows - 1) * ld + cols) * isz <= buf.nbytes, (off, rows, cols, ld, buf.nbytes)
    return np.ndarray((rows, cols), dtype=dt, buffer=buf, offset=off, strides=(ld * isz, isz))


def _local_product(kind: str, A: np.ndarray, B: np.ndarray) -> np.ndarray:
    if kind == "f64":
        return oracle.gemm_f64(np.ascontiguousarray(A), np.ascontiguousarray(B))
    if kind == "bf16":
        C, _ = oracle.gemm_bf16(np.ascontiguousarray(A), np.ascontiguousarray(B))
        return C.astype(np.float32)  # exact: the tests use exact-integer inputs
    C = oracle.gemm_s8(np.ascontiguousarray(A), np.ascontiguousarray(B))
    return C.astype(np.int32)


def comm_groups(plan_of_rank, world: int):
    """Create the gloo groups of every communicator kind; plan_of_rank(r) -> (steps, info).
    Returns {kind: (group, members)} for the calling rank (collective: all ranks call it)."""
    me = dist.get_rank()
    infos = [plan_of_rank(r)[1] for r in range(world)]
    out = {"WORLD": (None, list(range(world)))}
    for kind in ("ROW", "COL", "DEPTH"):
        colors = sorted({inf["color"][kind] for inf in infos if inf["color"][kind] >= 0})
        for c in colors:
            members = sorted((r for r in range(world) if infos[r]["color"][kind] == c),
                             key=lambda r: infos[r]["key"][kind])
            g = dist.new_group(members)  # every rank creates every group, in the same order
            if me in members:
                out[kind] = (g, members)
    return out


def execute(steps, info, kind: str, bufs: dict, groups: dict, cfull_bytes: int):
    """Run one rank's plan.  bufs: name -> np.uint8 array (A, B, C, CFULL on the root)."""
    me = dist.get_rank()
    bufs = dict(bufs)
    for i in range(4):
        if info["stage_bytes"][i] > 0:
            bufs[f"S{i}"] = np.zeros(info["stage_bytes"][i], np.uint8)
    peer_writes = []  # (offset, bytes) written into the root's C_full through CPEER
    pending = []

    def tens(name, off, n):
        return torch.from_numpy(bufs[name][off:off + n])

    def glob(comm, peer):
        return groups[comm][1][peer]

    for st in steps:
        op = st["op"]
        if op == "GEMM":
            dtin, dtout = IN_NP[kind], OUT_NP[kind]
            A = _view(bufs[st["src"]], st["src_off"], st["m"], st["n"], st["src_ld"], dtin)
            B = _view(bufs[st["src2"]], st["src2_off"], st["n"], st["p"], st["src2_ld"], dtin)
            C = _view(bufs[st["dst"]], st["dst_off"], st["m"], st["p"], st["dst_ld"], dtout)
            prod = _local_product(kind, A, B)
            if st["beta"]:
                C += prod
            else:
                C[...] = prod
            if st["dst"] == "CPEER" and groups["WORLD"][1] and bufs.get("CPEER") is not bufs.get("CFULL"):
                isz = np.dtype(dtout).itemsize
                for r in range(st["m"]):
                    o = st["dst_off"] + r * st["dst_ld"] * isz
                    peer_writes.append((o, bytes(bufs["CPEER"][o:o + st["p"] * isz])))
        elif op == "COPY2D":
            for r in range(st["m"]):
                d = st["dst_off"] + r * st["dst_ld"]
                s = st["src_off"] + r * st["src_ld"]
                bufs[st["dst"]][d:d + st["n"]] = bufs[st["src"]][s:s + st["n"]]
        elif op == "BCAST":
            g, mem = groups[st["comm"]]
            dist.broadcast(tens(st["dst"], st["dst_off"], st["n"]), src=mem[st["peer"]], group=g)
        elif op == "SEND":
            pending.append(dist.isend(tens(st["src"], st["src_off"], st["n"]), dst=glob(st["comm"], st["peer"])))
        elif op == "RECV":
            pending.append(dist.irecv(tens(st["dst"], st["dst_off"], st["n"]), src=glob(st["comm"], st["peer"])))
        elif op == "GROUP_START":
            pass
        elif op == "GROUP_END":
            for w in pending:
                w.wait()
            pending = []
        elif op == "REDUCE_SUM":
            g, mem = groups[st["comm"]]
            t = torch.from_numpy(bufs[st["dst"]][st["dst_off"]:st["dst_off"] + 8 * st["n"]].view(np.float64))
            root = mem[st["peer"]]
            dist.reduce(t if me == root else t.clone(), dst=root, group=g)  # NCCL: non-roots unchanged
        elif op == "MEMSET0":
            bufs[st["dst"]][st["dst_off"]:st["dst_off"] + st["n"]] = 0
        elif op == "BARRIER":
            # the fused gather's writes through the peer mapping land in the root's C_full
            if "CPEER" in bufs:
                allw = [None] * len(groups["WORLD"][1])
                dist.all_gather_object(allw, (me, peer_writes))
                if bufs.get("CFULL") is not None:
                    for (r, writes) in allw:
                        if r == me:
                            continue
                        for (o, data) in writes:
                            bufs["CFULL"][o:o + len(data)] = np.frombuffer(data, np.uint8)
            dist.barrier(group=groups[st["comm"]][0])
        elif op == "MAP_PEER":
            root = glob("WORLD", st["peer"])
            bufs["CPEER"] = bufs["CFULL"] if me == root else np.zeros(cfull_bytes, np.uint8)
        elif op in ("RECORD", "WAIT"):
            pass  # sequential execution in plan order
        else:
            raise AssertionError(f"unknown plan op {op}")
    return bufs


def _accesses(st, eo_in: int, eo_out: int):
    """(buffer, lo, hi, is_write) byte ranges a step touches."""
    op = st["op"]
    out = []
    if op == "GEMM":
        def span(off, rows, cols, ld, isz):
            return off, off + ((rows - 1) * ld + cols) * isz
        a = span(st["src_off"], st["m"], st["n"], st["src_ld"], eo_in)
        b = span(st["src2_off"], st["n"], st["p"], st["src2_ld"], eo_in)
        c = span(st["dst_off"], st["m"], st["p"], st["dst_ld"], eo_out)
        out += [(st["src"], *a, False), (st["src2"], *b, False), (st["dst"], *c, True)]
        if st["beta"]:
            out.append((st["dst"], *c, False))
    elif op == "COPY2D":
        out.append((st["src"], st["src_off"], st["src_off"] + (st["m"] - 1) * st["src_ld"] + st["n"], False))
        out.append((st["dst"], st["dst_off"], st["dst_off"] + (st["m"] - 1) * st["dst_ld"] + st["n"], True))
    elif op in ("BCAST", "RECV", "MEMSET0"):
        out.append((st["dst"], st["dst_off"], st["dst_off"] + st["n"], True))
        if op == "BCAST":
            out.append((st["dst"], st["dst_off"], st["dst_off"] + st["n"], False))
    elif op == "SEND":
        out.append((st["src"], st["src_off"], st["src_off"] + st["n"], False))
    elif op == "REDUCE_SUM":
        out.append((st["dst"], st["dst_off"], st["dst_off"] + 8 * st["n"], True))
    return out


def check_stream_order(steps, kind: str):
    """Assert the plan's two streams are race-free given its record/wait events (vector clocks)."""
    eo_in = np.dtype(IN_NP[kind]).itemsize
    eo_out = np.dtype(OUT_NP[kind]).itemsize
    clock = [[0, 0], [0, 0]]  # clock[s] = last index of each stream known to happen before stream s's next step
    events = {}
    history = []  # (stream, index-in-stream, accesses)
    count = [0, 0]
    for st in steps:
        s = st["stream"]
        if st["op"] == "RECORD":
            events[st["event"]] = list(clock[s])
            continue
        if st["op"] == "WAIT":
            assert st["event"] in events, f"wait on an event never recorded: {st}"
            clock[s] = [max(a, b) for a, b in zip(clock[s], events[st["event"]])]
            continue
        count[s] += 1
        clock[s][s] = count[s]
        acc = _accesses(st, eo_in, eo_out)
        for (s2, idx2, acc2) in history:
            if s2 == s:
                continue
            ordered = clock[s][s2] >= idx2
            for (b1, lo1, hi1, w1) in acc:
                for (b2, lo2, hi2, w2) in acc2:
                    if b1 == b2 and lo1 < hi2 and lo2 < hi1 and (w1 or w2):
                        assert ordered, f"race on {b1}[{lo1}:{hi1}] between stream {s2} step {idx2} and {st}"
        history.append((s, count[s], acc))
    # the caller's stream (0) must end after every step of the communication stream
    assert clock[0][1] >= count[1], "the caller's stream does not wait for the communication stream"
    # the communication stream must start after the caller's earlier work (buffers reused across calls)
    first1 = next((i for i, st in enumerate(steps) if st["stream"] == 1), None)
    if first1 is not None:
        assert steps[first1]["op"] == "WAIT", "the communication stream does not wait for the caller's stream first"
