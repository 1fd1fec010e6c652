L=paper_2408_15384_b200/libmm_b200.so
MM_F64_W16=1 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or fp64 or config1 or config2" 2>&1 | tail -2
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_W16=1 --cases f64:8192,f64:4096,f64:2000x1500x1750,f64:16384 --reps 6 2>&1 | tail -4
