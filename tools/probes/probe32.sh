timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or config0 or config1 or fixup" 2>&1 | tail -3
for s in f64:256 f64:300x200x520 f64:512; do MM_TRACE=1 timeout 120 python tools/one_case.py $s 4 2>&1 | grep "trace f64" | tail -1; done
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $B $L --cases f64:256,f64:300x200x520,f64:640x640x640 --reps 20 2>&1
timeout 600 python tools/overhead_probe.py --cases f64:256 2>&1
