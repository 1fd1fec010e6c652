"""Multi-rank mm_gemm_sharded over NCCL, one process per GPU (torchrun), on the CUDA path.

Runs tests/dist_nccl_worker.py under torchrun at G = 2, 4 and 8 when the box has that many GPUs
(skipped otherwise): the row-block layout of BASELINE.json configs[3] in every gather mode (incl.
MM_GATHER_C_FUSED's peer stores), SUMMA over the 1x2 / 2x2 / 2x4 grids of configs[4], and 2.5D
2x2x2 — at small ragged shapes bit-exact against the oracle, and at full size against SURVEY c7's
exact-integer checksums plus >= 64 sampled rows and columns of random inputs.  At G = 1 the same
worker runs on the one GPU (every layout degenerates to one rank), so the script itself is
exercised on every GPU run."""
import json
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _run(world, full, timeout):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={world}",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           os.path.join(ROOT, "tests", "dist_nccl_worker.py")] + (["--full"] if full else [])
    env = dict(os.environ, PYTHONPATH=ROOT)
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=timeout, env=env, cwd=ROOT)
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert lines, f"no result line (exit {out.returncode}):\n{out.stdout[-3000:]}\n{out.stderr[-3000:]}"
    res = json.loads(lines[-1])
    bad = [c for c in res["checks"] if not c.get("ok", True)]
    assert res["ok"] and not bad and out.returncode == 0, (bad, out.stderr[-2000:])
    return res


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_multi_rank(cuda_device, world):
    if torch.cuda.device_count() < world:
        pytest.skip(f"needs {world} GPUs, {torch.cuda.device_count()} visible")
    res = _run(world, full=True, timeout=3600)
    assert res["world"] == world


def test_sharded_worker_world1(cuda_device):
    res = _run(1, full=True, timeout=1800)
    assert res["world"] == 1 and len(res["checks"]) >= 20
