MM_F64_TILE=96 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or config1 or hand or edge" 2>&1 | tail -1
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_TILE=96 --cases f64:2000x1500x1750,f64:2048,f64:1536,f64:4096,f64:3000x2000x2500 --reps 10 2>&1 | tail -5
