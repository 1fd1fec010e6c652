set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
for E in MM_KA=1 MM_STREAMK=3 MM_STREAMK=0; do
echo "== B: $E"
timeout 600 python tools/ab_gpu.py $L $L --env-b $E --reps 20 --cases i8:4096,bf16:4096,i8:3072,bf16:2560,bf16:3072,i8:6144
done
} > $OUT/ab_r2zd.txt 2>&1
cat $OUT/ab_r2zd.txt
