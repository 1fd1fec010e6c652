set -u
OUT=gpurun_out; mkdir -p $OUT
for mc in 1 2; do for nt in 1 2; do for s in 8192 16384; do
MM_TRACE=1 MM_MC=$mc MM_NT=$nt timeout 120 python tools/one_case.py bf16:$s 3 2>&1 | grep "mm trace" | tail -1
done; done; done 2>&1 | tee $OUT/trace_mc.txt
