MM_KA=2 MM_NT=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "wide or guard" 2>&1 | tail -2
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_NT=2 --env-b MM_NT=2 MM_KA=2 --cases bf16:8192,bf16:16384,i8:8192,i8:4096 --reps 8 2>&1
for ka in 1 2; do MM_KA=$ka MM_NT=2 MM_TRACE=1 timeout 120 python tools/one_case.py bf16:16384 4 2>&1 | grep "clock\|mm trace\] m=" | tail -2 | sed "s/^/ka=$ka /"; done
