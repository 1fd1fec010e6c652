set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
# one round of 74 wide (256x512) pair tiles vs two rounds of 148 256x256 pair tiles, no tails
timeout 600 python tools/ab_gpu.py $L $L --env-a MM_NT=1 --env-b MM_NT=2 --reps 20 --cases i8:9472x4096x1024,i8:9472x8192x1024,bf16:9472x2048x1024,bf16:9472x4096x1024 > $OUT/ab_wide_round_r2zz23.txt 2>&1; cat $OUT/ab_wide_round_r2zz23.txt
