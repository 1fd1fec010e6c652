timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,bf16:2048,i8:2048,bf16:4096x4096x1024,bf16:8192,bf16:16384,bf16:3000x5000x4000 --reps 10 2>&1
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_STREAMK=2 --cases i8:4096,bf16:4096 --reps 10 2>&1
