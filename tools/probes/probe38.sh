L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_MC=2 MM_NT=1 --cases i8:4096,bf16:4096,i8:8192 --reps 12 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_MC=2 MM_NT=2 --cases i8:4096,bf16:4096 --reps 12 2>&1
for e in "MM_NT=2" "MM_MC=2 MM_NT=1"; do env $e MM_TRACE=1 timeout 120 python tools/one_case.py i8:4096 4 2>&1 | grep "timeline\|clock\|mm trace\] m=" | tail -3 | sed "s/^/$e /"; done
