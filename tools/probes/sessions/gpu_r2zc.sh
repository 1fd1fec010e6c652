set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
for P in 2 4 8; do
echo "== B: MM_L2_PF=$P"
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_L2_PF=$P --reps 20 --cases i8:4096,i8:3072,bf16:4096,bf16:8192,i8:8192,bf16:16384
done
} > $OUT/ab_r2zc.txt 2>&1
cat $OUT/ab_r2zc.txt
