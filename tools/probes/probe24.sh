for d in 0 2 1; do for s in bf16:16384; do
MM_DEBUG=$d MM_TRACE=1 timeout 120 python tools/one_case.py $s 6 2>&1 | grep "mm trace\] m=\|clock" | tail -2 | sed "s/^/debug=$d /"
done; done | tee gpurun_out/trace_clock2_r1.txt
for g in 4 8 16 32; do MM_GROUP_M=$g MM_TRACE=1 timeout 120 python tools/one_case.py bf16:16384 6 2>&1 | grep "mm trace\] m=\|clock" | tail -2 | sed "s/^/group=$g /"; done | tee -a gpurun_out/trace_clock2_r1.txt
