MM_F64_KB128=2 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or config1" 2>&1 | tail -1
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_KB128=2 --cases f64:8192,f64:4096,f64:2048,f64:16384 --reps 6 2>&1 | tail -4
