L=paper_2408_15384_b200/libmm_b200.so
MM_F64_W16=1 MM_F64_TILE=64 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or fp64" 2>&1 | tail -1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_TILE=128 --cases f64:640,f64:896,f64:1024,f64:1152 --reps 8 2>&1 | tail -4
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_W16=1 --cases f64:512,f64:640,f64:768,f64:896,f64:1024 --reps 8 2>&1 | tail -5
