set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
echo "== B: MM_EXP=1 (epilogue of tile j before the MMAs of tile j+1)"
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_EXP=1 --reps 30 --cases i8:4096,bf16:4096,i8:3072,bf16:2560,i8:8192
} > $OUT/ab_r2zg.txt 2>&1
cat $OUT/ab_r2zg.txt
