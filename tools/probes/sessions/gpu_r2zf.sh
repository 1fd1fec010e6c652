set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
echo "== B: MM_EPI_ST=1"
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_EPI_ST=1 --reps 30 --cases i8:4096,bf16:4096,i8:3072,bf16:2560,bf16:8192,i8:8192,bf16:16384
} > $OUT/ab_r2zf.txt 2>&1
cat $OUT/ab_r2zf.txt
MM_EPI_ST=1 timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q 2>&1 | tail -2
