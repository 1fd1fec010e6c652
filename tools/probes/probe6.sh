set -u
OUT=gpurun_out; mkdir -p $OUT
python tools/dbg_f64.py 128
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_fix.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu_fix.log
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases f64:256,f64:512,f64:2000x1500x1750 --reps 10 2>&1 | tee $OUT/ab_f64b.txt
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_NT=2 --cases i8:4096,bf16:4096,i8:2048,bf16:2048 --reps 10 2>&1 | tee $OUT/ab_nt2_small.txt
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_NT=2 MM_STREAMK=1 --cases i8:4096,bf16:4096,i8:2048,bf16:2048 --reps 10 2>&1 | tee -a $OUT/ab_nt2_small.txt
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_STREAMK=1 --cases i8:4096,bf16:4096 --reps 10 2>&1 | tee -a $OUT/ab_nt2_small.txt
