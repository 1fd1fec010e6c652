timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -x -q -k "tc or fuzz or reduce or config2 or split" 2>&1 | tail -1
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,bf16:1024,bf16:256,i8:8192 --reps 12 2>&1 | tail -5
