OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_r1r.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_gpu_r1r.log
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,i8:8192,bf16:8192,bf16:16384 --reps 10 2>&1 | tee $OUT/ab_r1r.txt
for nt in 2; do for s in i8:4096 bf16:16384; do MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "mm trace" | tail -1; done; done | tee $OUT/trace_r1r.txt
