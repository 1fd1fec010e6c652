MM_KA=2 MM_NT=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tc or tiny or handworked or fixup or random or identity or guard or config2 or stream_k" 2>&1 | tail -2
for ka in 1 2; do for d in 1 0; do MM_KA=$ka MM_DEBUG=$d MM_NT=1 MM_TRACE=1 timeout 120 python tools/one_case.py i8:4096 4 2>&1 | grep "timeline\|clock" | tail -2 | sed "s/^/ka=$ka debug=$d /"; done; done
L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $L $L --env-a MM_NT=1 --env-b MM_NT=1 MM_KA=2 --cases i8:4096,bf16:4096,bf16:8192,i8:8192 --reps 10 2>&1
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_NT=1 MM_KA=2 --cases i8:4096,bf16:4096,bf16:8192,bf16:16384 --reps 10 2>&1
