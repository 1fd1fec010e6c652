set -u
OUT=gpurun_out
L=paper_2408_15384_b200
timeout 900 python tools/ab_gpu.py $L/libmm_b200_base.so $L/libmm_b200.so --reps 16 --cases i8:4096,i8:8192,i8:16384,bf16:8192 > $OUT/ab_i8_batchcode_r2zz17.txt 2>&1; cat $OUT/ab_i8_batchcode_r2zz17.txt
timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 8192 8192 16384 > $OUT/ab_emu_repeat_r2zz17.txt 2>&1; cat $OUT/ab_emu_repeat_r2zz17.txt
