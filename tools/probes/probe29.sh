OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_epi8.log 2>&1; echo "pytest rc=$?"; tail -3 $OUT/pytest_epi8.log
for s in i8:4096 bf16:16384; do MM_TRACE=1 timeout 120 python tools/one_case.py $s 3 2>&1 | grep "timeline\|per 4-KB\|clock\|mm trace\] m=" | tail -4; done | tee $OUT/trace_epi8.txt
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,i8:8192,bf16:8192,bf16:2048,bf16:16384 --reps 10 2>&1 | tee $OUT/ab_epi8.txt
