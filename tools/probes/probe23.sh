for d in 0 1; do for s in bf16:16384; do
MM_DEBUG=$d MM_TRACE=1 timeout 120 python tools/one_case.py $s 6 2>&1 | grep "mm trace\] m=\|clock" | tail -2 | sed "s/^/debug=$d /"
done; done | tee gpurun_out/trace_clock_r1.txt
