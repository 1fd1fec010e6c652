OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tail_subtiles" > $OUT/pytest_tsplit.log 2>&1; echo "pytest tsplit rc=$?"; tail -3 $OUT/pytest_tsplit.log
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,i8:2100x640x3000,bf16:16384 --reps 10 2>&1 | tee $OUT/ab_tsplit.txt
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_TSPLIT=2 --cases i8:4096,bf16:4096 --reps 10 2>&1 | tee -a $OUT/ab_tsplit.txt
