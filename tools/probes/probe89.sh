timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "f64 or config0 or hand or fuzz or brute or edge" 2>&1 | tail -2
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 300 python tools/ab_gpu.py $B $L --cases f64:256,f64:256x512x256,f64:192,f64:320,f64:128 --reps 20 2>&1 | tail -5
FLUSH=1 MM_TRACE=1 timeout 120 python tools/one_case.py f64:256 4 2>&1 | grep "mm trace f64" | tail -1
