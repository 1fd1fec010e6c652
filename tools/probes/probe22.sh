for d in 0 1; do for nt in 1 2; do for s in i8:4096 bf16:8192 bf16:16384; do
MM_DEBUG=$d MM_NT=$nt MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "mm trace\] m=" | tail -1 | sed "s/^/debug=$d /"
done; done; done | tee gpurun_out/trace_noload_r1.txt
