OUT=gpurun_out
MM_EPI_BOX=0 timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "not f64 and not config4 and not config0 and not config1" > $OUT/pytest_box0.log 2>&1; echo "pytest box0 rc=$?"; tail -2 $OUT/pytest_box0.log
for b in 32 0; do for s in i8:4096 bf16:8192 bf16:16384; do MM_EPI_BOX=$b MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "mm trace" | tail -3 | sed "s/^/box$b /"; done; done | tee $OUT/trace_box0.txt
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_EPI_BOX=0 --cases i8:4096,bf16:4096,i8:8192,bf16:8192,bf16:2048,bf16:16384 --reps 10 2>&1 | tee $OUT/ab_box0.txt
