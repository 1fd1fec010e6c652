# r2c: FP64 producer-less kernel — parity (fp64 tests + fuzz) and A/B vs the producer-warp kernel
set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_hazards.py -q -x -k "f64 or fuzz or split or held or streams" > $OUT/pytest_r2c.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_r2c.log; tail -3 $OUT/pytest_r2c.log
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_PRODUCER=1 --cases f64:2000x1500x1750,f64:4096,f64:8192,f64:16384,f64:3000x5000x4000,f64:1536 --reps 10 > $OUT/ab_f64pl_r2c.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_B2D=1 --cases f64:2000x1504x1760,f64:8192 --reps 10 >> $OUT/ab_f64pl_r2c.txt 2>&1
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_F64_PRODUCER=1 --cases f64:32768 --reps 3 >> $OUT/ab_f64pl_r2c.txt 2>&1
cat $OUT/ab_f64pl_r2c.txt
