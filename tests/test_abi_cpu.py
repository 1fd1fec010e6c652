"""C-ABI checks that need no GPU: the library loads, exports every symbol
include/mm.h declares, the pure host functions (partition rule, SUMMA panel
schedule, status strings) behave, and the product path refuses to run without a
device instead of falling back to the CPU."""
import ctypes
import os
import re
import subprocess

import pytest
import torch

import paper_2408_15384_b200 as mm
from paper_2408_15384_b200 import _lib

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def declared_symbols():
    with open(os.path.join(ROOT, "include", "mm.h")) as f:
        src = f.read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(mm_[a-z_0-9]+)\s*\(", src)))


def test_header_declares_what_binding_expects():
    assert declared_symbols() == sorted(_lib.EXPORTS)


def test_library_exports_every_declared_symbol():
    lib = _lib.load()
    for name in declared_symbols():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True, text=True, check=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared_symbols()) <= exported
    # internal symbols stay hidden (-fvisibility=hidden)
    assert not any(s.startswith("_ZN3mmb") for s in exported)


def test_library_is_sm100a_sass():
    out = subprocess.run(["cuobjdump", "-lelf", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out
    sass = subprocess.run(["cuobjdump", "-sass", _lib.LIB_PATH], capture_output=True, text=True).stdout
    for mnemonic in ("UTCHMMA", "UTCIMMA", "UTMALDG", "LDTM", "DMMA"):
        assert mnemonic in sass, mnemonic


def test_version_and_status_strings():
    assert "sm_100a" in mm.version()
    lib = _lib.load()
    assert lib.mm_status_string(0) == b"MM_OK"
    assert lib.mm_status_string(2) == b"MM_ERR_USAGE"
    assert lib.mm_status_string(99) == b"MM_ERR_UNKNOWN"
    assert lib.mm_last_error(None) == b"NULL context"


def test_null_context_is_usage_error():
    lib = _lib.load()
    assert lib.mm_gemm(None, 4, 4, 4, 0, 1, 2, 3, None) == _lib.MM_ERR_USAGE
    assert lib.mm_sync_check(None, None) == _lib.MM_ERR_USAGE
    assert lib.mm_create(0, None, 0, None) == _lib.MM_ERR_USAGE
    lib.mm_destroy(None)  # no-op


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU refusal")
def test_no_gpu_refuses_instead_of_falling_back():
    h = ctypes.c_void_p()
    st = _lib.load().mm_create(0, None, 0, ctypes.byref(h))
    assert st == _lib.MM_ERR_UNSUPPORTED and not h.value
    with pytest.raises(mm.MMError):
        mm.Context(0)


# ---------------------------------------------------------------- partition rule
@pytest.mark.parametrize("total", [1, 2, 7, 8, 9, 100, 16384, 2000])
@pytest.mark.parametrize("G", [1, 2, 3, 4, 8, 16])
def test_shard_range_partition(total, G):
    q = -(-total // G)
    covered = []
    for r in range(G):
        s, c = mm.shard_range(total, G, r)
        assert c >= 0
        if c:
            covered.extend(range(s, s + c))
            assert c == q or s + c == total  # all full except the last non-empty one
    assert covered == list(range(total))  # contiguous, ordered, disjoint, complete


def test_shard_range_surplus_workers_empty():
    assert [mm.shard_range(3, 8, r)[1] for r in range(8)] == [1, 1, 1, 0, 0, 0, 0, 0]
    assert mm.shard_range(10, 4, 3) == (9, 1)  # ⌈10/4⌉=3: 3,3,3,1
    assert mm.shard_range(5, 2, 5) == (0, 0)   # r outside [0, G)


@pytest.mark.parametrize("n,pr,pc,panel", [(32768, 2, 4, 2048), (1000, 2, 3, 64), (7, 4, 2, 2), (5, 1, 1, 100),
                                           (1500, 3, 2, 256), (3, 4, 4, 1)])
def test_summa_panels_cover_and_respect_blocks(n, pr, pc, panel):
    panels = mm.summa_panels(n, pr, pc, panel)
    k = 0
    for (k0, kw, ao, bo) in panels:
        assert k0 == k and 1 <= kw <= panel
        s, c = mm.shard_range(n, pc, ao)  # A column block owning the panel
        assert s <= k0 and k0 + kw <= s + c
        s, c = mm.shard_range(n, pr, bo)  # B row block owning the panel
        assert s <= k0 and k0 + kw <= s + c
        k += kw
    assert k == n


def test_workspace_size_bound():
    """mm_workspace_size through the C-ABI: 0 for invalid arguments; at least the
    zero-padded operand copies of the edge path; grows with the shape; the sharded layouts add
    their panel staging (G > 1) — pure host logic, no device."""
    lib = _lib.load()
    f = lib.mm_workspace_size
    assert f(0, 4, 4, 0, 0, 1) == 0 and f(4, 4, 4, 7, 0, 1) == 0 and f(4, 4, 4, 0, 9, 1) == 0
    assert f(4, 4, 4, 1, 1, 2) == 0  # SUMMA layouts are FP64 only
    for dt, esz in ((0, 8), (1, 2), (2, 1)):
        small, big = f(300, 200, 100, dt, 0, 1), f(3000, 2000, 1000, dt, 0, 1)
        assert small > 0 and big > small
        al = 16 // esz
        pad = (3000 * (-(-2000 // al) * al) + 2000 * (-(-1000 // al) * al)) * esz
        assert big >= pad
    # row-block with G ranks: the B broadcast stages two column panels of B (p/8 wide each)
    n, p = 4096, 4096
    assert f(4096, n, p, 1, 0, 8) >= 2 * n * (p // 8) * 2
    # SUMMA: two panel sets, the largest over the grids G factors into
    assert f(8192, 8192, 8192, 0, 1, 8) >= 2 * (8192 * 2048 * 8)
    assert mm.workspace_size(16384, 16384, 16384, torch.bfloat16) == f(16384, 16384, 16384, 1, 0, 1)


def test_diag_knobs_refused_by_release_build(monkeypatch):
    """MM_DEBUG (skips loads/stores: garbage results) and MM_TRACE / MM_HOST_TRACE (hidden stream
    synchronisations) exist only in the diagnostic build; the release library refuses them with
    MM_ERR_UNSUPPORTED before touching the device.  Checked here on the release .so's strings and in
    tests/test_gpu_parity.py on the device."""
    out = subprocess.run(["strings", _lib.LIB_PATH], capture_output=True, text=True).stdout
    assert "is a diagnostic knob of the diagnostic build only" in out
    assert "[mm trace]" not in out  # the timeline printers are compiled out of the release library


def test_f64_emu_plan():
    """mm_f64_emu_plan (MM_F64_EMU's host plan, csrc/f64_emu.cu) checked with exact integers: the
    moduli are pairwise coprime and ≤ 256 (residues fit INT8), the scaled integer product fits the
    symmetric CRT range (n·2^(2β) ≤ M/2 − 1, so Chinese remaindering recovers it exactly), β ≥ 53
    (the binary64 width of every row / column maximum), β is the largest the product allows (≤ 60),
    and no shorter prefix of the list would give β ≥ 53; INT32 sums bound n (n·2^14 < 2^31)."""
    import math
    lib = _lib.load()
    mods, cnt, beta = (ctypes.c_int * 16)(), ctypes.c_int(), ctypes.c_int()
    full = None
    for n in (1, 2, 7, 8, 9, 100, 1000, 1500, 2049, 4096, 32768, 65536, 131071):
        assert lib.mm_f64_emu_plan(n, mods, ctypes.byref(cnt), ctypes.byref(beta)) == _lib.MM_OK, n
        c, b = cnt.value, beta.value
        ms = list(mods[:c])
        if full is None or len(ms) > len(full):
            full = ms
        assert all(2 <= x <= 256 for x in ms)
        assert all(math.gcd(x, y) == 1 for i, x in enumerate(ms) for y in ms[:i])
        M = math.prod(ms)
        assert n * 2 ** (2 * b) <= M // 2 - 1, (n, c, b)
        assert b >= 53
        assert b == 60 or n * 2 ** (2 * (b + 1)) > M // 2 - 1, (n, b)  # β maximal
        Mless = math.prod(ms[:-1])
        assert n * 2 ** (2 * 53) > Mless // 2 - 1, (n, c)  # the fewest moduli
        assert n * (128 * 128) < 2 ** 31  # exact INT32 sums of residue products
    # every plan uses a prefix of one fixed list
    for n in (1, 1000, 131071):
        assert lib.mm_f64_emu_plan(n, mods, ctypes.byref(cnt), ctypes.byref(beta)) == _lib.MM_OK
        assert list(mods[:cnt.value]) == full[:cnt.value]
    assert lib.mm_f64_emu_plan(131072, mods, ctypes.byref(cnt), ctypes.byref(beta)) == _lib.MM_ERR_UNSUPPORTED
    assert lib.mm_f64_emu_plan(0, mods, ctypes.byref(cnt), ctypes.byref(beta)) == _lib.MM_ERR_USAGE
    assert lib.mm_f64_emu_plan(5, None, ctypes.byref(cnt), ctypes.byref(beta)) == _lib.MM_OK
    assert lib.mm_f64_emu_plan(5, None, None, ctypes.byref(beta)) == _lib.MM_ERR_USAGE
    # workspace: residue planes of A, B and C + the INT32 product (+ the INT8 product's own)
    f = lib.mm_workspace_size
    m, n, p = 2000, 1500, 1750
    assert lib.mm_f64_emu_plan(n, mods, ctypes.byref(cnt), ctypes.byref(beta)) == _lib.MM_OK
    assert f(m, n, p, 3, 0, 1) >= cnt.value * (m * n + n * p + m * p) + 4 * m * p
    assert f(m, 131072, p, 3, 0, 1) == 0 and f(m, n, p, 3, 0, 2) >= f(m, n, p, 3, 0, 1) // 2  # sharded: local products
