for s in i8:4096 bf16:8192 bf16:16384; do MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "mm trace" | tail -2; done | tee gpurun_out/trace_r1v.txt
