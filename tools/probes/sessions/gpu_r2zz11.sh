set -u
OUT=gpurun_out
L=paper_2408_15384_b200
timeout 1200 python tools/ab_gpu.py $L/libmm_b200_base.so $L/libmm_b200.so --reps 16 --cases bf16:16384,bf16:8192,bf16:4096,i8:4096,i8:8192,f64:8192,f64:2000x1500x1750,f64:256 > $OUT/ab_session_r2zz11.txt 2>&1; cat $OUT/ab_session_r2zz11.txt
