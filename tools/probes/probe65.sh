timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "reduce_add or stream_k or wide_tiles or fixup_repeated" 2>&1 | tail -4
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,i8:3072,bf16:3072,i8:2560,bf16:2560,i8:6144,bf16:6144 --reps 10 2>&1 | tail -8
