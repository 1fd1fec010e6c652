set -u
OUT=gpurun_out
L=paper_2408_15384_b200
{
timeout 900 python tools/ab_gpu.py $L/libmm_b200_base.so $L/libmm_b200.so --reps 20 --cases i8:4096x4096x8192,i8:7168,bf16:7168,i8:6144,bf16:6144,i8:8192,bf16:8192,i8:4096,bf16:4096,i8:3072x8192x5120,bf16:5120x4096x6144,i8:2048x4096x16384,bf16:16384
} > $OUT/ab_r2zj.txt 2>&1
cat $OUT/ab_r2zj.txt
