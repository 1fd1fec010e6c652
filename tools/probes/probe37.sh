timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_NO_B3=1 --cases bf16:4096,bf16:8192,bf16:16384,bf16:2048,bf16:4096x4096x1024 --reps 10 2>&1
for e in "MM_NO_B3=1" "MM_NO_B3="; do env $e MM_TRACE=1 timeout 120 python tools/one_case.py bf16:16384 4 2>&1 | grep "clock\|mm trace\] m=" | tail -2 | sed "s/^/$e /"; done
