set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
MM_F64_TILE=9612 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "f64" > $OUT/pytest_r2t.log 2>&1; echo "pytest rc=$?"; tail -1 $OUT/pytest_r2t.log
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_TILE=9612 --cases f64:2000x1500x1750,f64:4096,f64:8192,f64:16384 --reps 8 > $OUT/ab_f64w12_r2t.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_TILE=9612 --cases f64:32768 --reps 2 >> $OUT/ab_f64w12_r2t.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_TILE=96 --env-b MM_F64_TILE=9612 --cases f64:8192,f64:2000x1500x1750 --reps 8 >> $OUT/ab_f64w12_r2t.txt 2>&1
cat $OUT/ab_f64w12_r2t.txt
