B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases f64:8192,f64:4096,f64:2000x1500x1750,f64:1024 --reps 8 2>&1 | tail -4
