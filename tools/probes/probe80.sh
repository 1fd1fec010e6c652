MM_KA=1 MM_DEBUG=32 timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tc_ or config2 or tiny" 2>&1 | tail -1
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_KA=1 --env-b MM_KA=1 MM_DEBUG=32 --cases i8:4096,bf16:4096,i8:8192 --reps 8 2>&1 | tail -3
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_KA=1 MM_DEBUG=32 --cases i8:4096,bf16:4096,i8:8192 --reps 8 2>&1 | tail -3
