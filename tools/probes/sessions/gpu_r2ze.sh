set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200_diag.so
{
for E in MM_DEBUG=4 MM_DEBUG=28 MM_DEBUG=1; do
echo "== B: $E"
timeout 600 python tools/ab_gpu.py $L $L --env-b $E --reps 30 --cases i8:4096,bf16:4096,bf16:8192
done
} > $OUT/ab_r2ze.txt 2>&1
cat $OUT/ab_r2ze.txt
