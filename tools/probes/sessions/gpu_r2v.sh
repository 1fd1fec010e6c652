set -u
OUT=gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_gpu_hazards.py tests/test_gpu_sharded.py -q -x > $OUT/pytest_r2v.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_r2v.log
timeout 900 python tools/variants_ab.py f64:2000x1500x1750 --flush --reps 20 --rounds 3 --variants "base" > $OUT/var_f64_r2v.txt 2>&1
timeout 900 python tools/variants_ab.py f64:32768 --window-s 4 --rounds 1 --variants "base" >> $OUT/var_f64_r2v.txt 2>&1
cat $OUT/var_f64_r2v.txt
