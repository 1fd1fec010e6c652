set -u
OUT=gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $OUT/smi_r2y.txt
timeout 900 python tools/ab_gpu.py paper_2408_15384_b200/libmm_b200_base.so paper_2408_15384_b200/libmm_b200.so --reps 20 \
  --cases i8:4096,bf16:4096,i8:2560,bf16:2560,i8:3072,bf16:2048,i8:8192,bf16:8192,bf16:16384,i8:2000x12288x3000 > $OUT/ab_r2y.txt 2>&1
cat $OUT/ab_r2y.txt
timeout 900 python -m pytest tests -m gpu -x -q > $OUT/pytest_r2y.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_r2y.log
tail -3 $OUT/pytest_r2y.log
