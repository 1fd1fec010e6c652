set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
echo "== B: MM_EXP=2 (all of A and B prefetched into L2 at start)"
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_EXP=2 --reps 30 --cases i8:4096,bf16:4096,i8:3072,bf16:3072,i8:2048,bf16:2048,i8:5120,i8:4096x4096x8192
} > $OUT/ab_r2zk.txt 2>&1
cat $OUT/ab_r2zk.txt
