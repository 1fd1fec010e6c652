L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_STREAMK=0 --cases bf16:2048x16384x16384,bf16:4096x16384x16384,bf16:8192x16384x16384 --reps 8 2>&1 | tail -3
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_NT=1 --cases bf16:2048x16384x16384,bf16:4096x16384x16384 --reps 8 2>&1 | tail -2
