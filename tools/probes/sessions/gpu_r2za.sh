set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
echo "== B: MM_TMA_STORE=0 (register stores)"
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_TMA_STORE=0 --reps 20 --cases i8:4096,bf16:4096,i8:3072,i8:8192,bf16:8192
echo "== B: MM_NT=2"
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_NT=2 --reps 20 --cases i8:4096,i8:3072
} > $OUT/ab_r2za.txt 2>&1
cat $OUT/ab_r2za.txt
