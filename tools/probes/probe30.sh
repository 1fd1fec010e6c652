OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_pdl.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_pdl.log
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_NO_PDL=1 --cases f64:256,f64:2000x1500x1750,i8:4096,bf16:4096,bf16:16384 --reps 12 2>&1 | tee $OUT/ab_pdl.txt
timeout 600 python tools/overhead_probe.py --cases f64:256,bf16:4096,i8:4096 2>&1 | tee $OUT/overhead_pdl.txt
MM_NO_PDL=1 timeout 600 python tools/overhead_probe.py --cases f64:256,bf16:4096,i8:4096 2>&1 | tee -a $OUT/overhead_pdl.txt
