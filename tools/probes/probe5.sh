set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_gpu_f64.log 2>&1; echo "pytest rc=$?"; tail -4 $OUT/pytest_gpu_f64.log
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases f64:256,f64:512,f64:1024,f64:2000x1500x1750,f64:4096,f64:8192,f64:16384 --reps 8 2>&1 | tee $OUT/ab_f64.txt
