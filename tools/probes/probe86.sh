MM_F64_KS=42 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "config0 or hand or f64_tiles" 2>&1 | tail -1
L=paper_2408_15384_b200/libmm_b200.so
timeout 300 python tools/ab_gpu.py $L $L --env-b MM_F64_KS=42 --cases f64:256,f64:256x512x256,f64:192,f64:320 --reps 20 2>&1 | tail -4
python - <<'PY'
import os, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2408_15384_b200 as mm
A = torch.rand(256, 256, dtype=torch.float64, device="cuda"); B = torch.rand(256, 256, dtype=torch.float64, device="cuda")
C = torch.empty(256, 256, dtype=torch.float64, device="cuda")
def graph_us(f, n=100):
    f(); torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):
        for _ in range(n): f()
    ts = []
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); g.replay(); e1.record(); e1.synchronize(); ts.append(e0.elapsed_time(e1) * 1e3 / n)
    return min(ts)
for ks in ("", "42"):
    if ks: os.environ["MM_F64_KS"] = ks
    else: os.environ.pop("MM_F64_KS", None)
    print("KS", ks or "default", f"{graph_us(lambda: mm.gemm(A, B, out=C)):.2f} us/launch in a graph")
PY
