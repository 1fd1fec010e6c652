for s in f64:256 f64:2000x1500x1750; do MM_TRACE=1 timeout 120 python tools/one_case.py $s 4 2>&1 | grep "trace f64" | tail -1; done | tee gpurun_out/f64_timeline_r1.txt
