set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
cat > /tmp/emu_knob_ab.py <<'PY'
import os, statistics, sys, torch
sys.path.insert(0, os.getcwd())
import paper_2408_15384_b200 as mm
def t(fn, reps):
    fn(); torch.cuda.synchronize(); ts=[]
    for _ in range(reps):
        a,b=torch.cuda.Event(True),torch.cuda.Event(True); a.record(); fn(); b.record(); b.synchronize(); ts.append(a.elapsed_time(b))
    return statistics.fmean(ts)
for N in (3072, 4096, 6144, 8192):
    A=torch.rand(N,N,dtype=torch.float64,device="cuda"); B=torch.rand(N,N,dtype=torch.float64,device="cuda"); C=torch.empty_like(A)
    res={}
    for rnd in range(2):
        for v in (["0","1","1g4"] if rnd == 0 else ["1g4","1","0"]):
            os.environ["MM_EMU_BATCH"]=v[0]
            if v.endswith("g4"): os.environ["MM_GROUP_M"]="4"
            res.setdefault(v,[]).append(t(lambda: mm.gemm(A,B,out=C,f64_emulation=True), 6))
            os.environ.pop("MM_GROUP_M",None)
    print(N, {k: round(statistics.fmean(v),3) for k,v in res.items()}, flush=True)
PY
timeout 900 python /tmp/emu_knob_ab.py > $OUT/ab_emu_batch_knob_r2zz20.txt 2>&1; cat $OUT/ab_emu_batch_knob_r2zz20.txt
