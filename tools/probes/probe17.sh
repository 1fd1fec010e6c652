OUT=gpurun_out
MM_EPI_BOX=128 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "not f64" > $OUT/pytest_box128.log 2>&1; echo "pytest box128 rc=$?"; tail -2 $OUT/pytest_box128.log
for b in 32 128; do for s in i8:4096 bf16:8192 bf16:16384; do MM_EPI_BOX=$b MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "mm trace" | tail -2 | sed "s/^/box$b /"; done; done | tee $OUT/trace_r1w.txt
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_EPI_BOX=128 --cases i8:4096,bf16:4096,i8:8192,bf16:8192,bf16:2048,bf16:16384 --reps 10 2>&1 | tee $OUT/ab_r1w.txt
