set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
for E in MM_EXP=8 MM_EXP=16; do
echo "== B: $E (consumer warps in step every 1 / 4 k-blocks)"
timeout 900 python tools/ab_gpu.py $L $L --env-b $E --reps 10 --cases f64:8192,f64:4096,f64:2000x1500x1750
done
} > $OUT/ab_r2zq.txt 2>&1
cat $OUT/ab_r2zq.txt
