set -u
OUT=gpurun_out
L=paper_2408_15384_b200
for i in 1 2; do
timeout 600 python tools/ab_gpu.py $L/libmm_b200_base.so $L/libmm_b200.so --reps 40 --cases bf16:16384,i8:4096,bf16:12288
timeout 600 python tools/ab_gpu.py $L/libmm_b200.so $L/libmm_b200_base.so --reps 40 --cases bf16:16384,i8:4096,bf16:12288
done > $OUT/ab_r2z.txt 2>&1
cat $OUT/ab_r2z.txt
