set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
echo "== B: MM_EXP=4 (FP64 consumer release without the proxy fence; timing only)"
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_EXP=4 --reps 10 --cases f64:8192,f64:4096,f64:2000x1500x1750
} > $OUT/ab_r2zo.txt 2>&1
cat $OUT/ab_r2zo.txt
