python - <<'PY'
import os, sys, time, torch
sys.path.insert(0, os.getcwd())
import paper_2408_15384_b200 as mm
N=16384
A = torch.randn(N, N).to(torch.bfloat16).pin_memory()
B = torch.randn(N, N).to(torch.bfloat16).pin_memory()
C = torch.empty(N, N, dtype=torch.float32).pin_memory()
mm.gemm_host(A, B, out=C); mm.gemm_host(A, B, out=C)
os.environ["MM_HOST_TRACE"]="1"
mm.gemm_host(A, B, out=C)
del os.environ["MM_HOST_TRACE"]
# raw copy rates: contiguous 512 MB H2D, D2H, both at once
dA = torch.empty_like(A, device="cuda"); dC = torch.empty_like(C, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(f):
    torch.cuda.synchronize(); t0=time.perf_counter(); f(); torch.cuda.synchronize(); return time.perf_counter()-t0
for _ in range(2): t(lambda: dA.copy_(A, non_blocking=True))
h2d = t(lambda: dA.copy_(A, non_blocking=True)); d2h = t(lambda: C.copy_(dC, non_blocking=True))
def both():
    with torch.cuda.stream(s1): dA.copy_(A, non_blocking=True)
    with torch.cuda.stream(s2): C[:N//2].copy_(dC[:N//2], non_blocking=True)
tb = t(both)
print(f"H2D 512MB {h2d*1e3:.1f} ms = {A.numel()*2/h2d/1e9:.1f} GB/s; D2H 1GB {d2h*1e3:.1f} ms = {C.numel()*4/d2h/1e9:.1f} GB/s; both (512MB each way) {tb*1e3:.1f} ms = {2*A.numel()*2/tb/1e9:.1f} GB/s")
PY
