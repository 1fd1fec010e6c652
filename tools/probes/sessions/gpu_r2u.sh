set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
for T in 12896 96192; do MM_F64_TILE=$T timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "f64" > $OUT/pytest_r2u_$T.log 2>&1; echo "pytest $T rc=$?"; tail -1 $OUT/pytest_r2u_$T.log; done
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_TILE=9612 --env-b MM_F64_TILE=12896 --cases f64:2000x1500x1750,f64:8192,f64:16384 --reps 8 > $OUT/ab_f64w12b_r2u.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_TILE=9612 --env-b MM_F64_TILE=96192 --cases f64:2000x1500x1750,f64:8192,f64:16384 --reps 8 >> $OUT/ab_f64w12b_r2u.txt 2>&1
cat $OUT/ab_f64w12b_r2u.txt
