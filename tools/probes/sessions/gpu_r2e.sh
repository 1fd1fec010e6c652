# r2e: FP64 several CTAs per SM (MM_F64_CPS=2/3): parity + A/B vs one 16-warp CTA per SM
set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
for v in 2 3; do MM_F64_CPS=$v timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "f64" > $OUT/pytest_r2e_cps$v.log 2>&1; echo "cps$v pytest rc=$?"; tail -1 $OUT/pytest_r2e_cps$v.log; done
timeout 600 python -m pytest tests/test_gpu_fuzz.py -q -x > $OUT/pytest_r2e_fuzz.log 2>&1; echo "fuzz rc=$?"; tail -1 $OUT/pytest_r2e_fuzz.log
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_CPS=2 --cases f64:2000x1500x1750,f64:4096,f64:8192,f64:16384 --reps 8 > $OUT/ab_f64cps_r2e.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_CPS=3 --cases f64:2000x1500x1750,f64:4096,f64:8192,f64:16384 --reps 8 >> $OUT/ab_f64cps_r2e.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_CPS=2 --cases f64:32768 --reps 2 >> $OUT/ab_f64cps_r2e.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-b MM_F64_CPS=3 --cases f64:32768 --reps 2 >> $OUT/ab_f64cps_r2e.txt 2>&1
cat $OUT/ab_f64cps_r2e.txt
