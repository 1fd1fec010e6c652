L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_TILE=128 --cases f64:1024,f64:1280,f64:1536,f64:1792,f64:2048,f64:3000x1000x2000,f64:768 --reps 8 2>&1 | tail -7
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_TILE=64 --cases f64:2048,f64:2000x1500x1750 --reps 8 2>&1 | tail -2
