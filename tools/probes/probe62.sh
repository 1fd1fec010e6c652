L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or fp64 or config1 or config2" 2>&1 | tail -1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_TILE=128 --cases f64:1024,f64:1152,f64:1280,f64:1408,f64:1536,f64:1000x3000x1500 --reps 8 2>&1 | tail -6
