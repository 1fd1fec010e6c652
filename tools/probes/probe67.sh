B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,i8:2560,bf16:2560,bf16:7680,i8:7680,bf16:2000x8192x3000,i8:2000x12288x3000,bf16:5120 --reps 10 2>&1 | tail -9
