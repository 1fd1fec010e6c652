OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or fixup or config0 or config1" > $OUT/pytest_f64ks.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_f64ks.log
for st in 1 0; do for s in i8:4096 bf16:8192 bf16:16384; do MM_TMA_STORE=$st MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "mm trace" | tail -1 | sed "s/^/tma_store=$st /"; done; done | tee $OUT/trace_r1s.txt
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $B $L --cases f64:256,f64:300x200x520 --reps 20 2>&1 | tee $OUT/ab_r1s.txt
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_TMA_STORE=0 --cases i8:4096,bf16:4096,bf16:8192 --reps 10 2>&1 | tee -a $OUT/ab_r1s.txt
