timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or config0 or config1 or fixup or tiny" 2>&1 | tail -3
for kb in 1 4; do MM_F64_KB=$kb MM_TRACE=1 timeout 120 python tools/one_case.py f64:256 4 2>&1 | grep "trace f64" | tail -1 | sed "s/^/kb=$kb /"; done
L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $L $L --env-a MM_F64_KB=1 --cases f64:256,f64:512x256x512 --reps 20 2>&1
timeout 600 python tools/overhead_probe.py --cases f64:256 2>&1
