L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $L $L --env-a MM_NT=2 --env-b MM_NT=1 --cases bf16:2048x16384x16384,bf16:4096x16384x16384,bf16:8192x16384x16384 --reps 8 2>&1 | tee gpurun_out/ab_shard_nt_r1y.txt
