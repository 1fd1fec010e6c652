L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_STREAMK=0 --cases bf16:256,bf16:256x2048x256,bf16:512x1536x512,bf16:1024,bf16:1024x4096x1024,bf16:2560,i8:512x8192x512,i8:1024x8192x1024,bf16:1536,bf16:2048 --reps 10 2>&1 | tail -10
