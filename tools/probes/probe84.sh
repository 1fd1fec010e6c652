timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "f64 or config1 or config0 or fuzz or hand" 2>&1 | tail -1
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases f64:2000x1500x1750,f64:2048,f64:1536,f64:4096,f64:8192,f64:256 --reps 10 2>&1 | tail -6
