timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "i8 or config2 or fuzz or tc" 2>&1 | tail -1
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,i8:3072,i8:6144,i8:8192,i8:2560,i8:5120,i8:3000x5000x4000 --reps 16 2>&1 | tail -7
