# r2n: N-half tail tiles (MM_STREAMK=4): parity + timing
set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "n_half_tail" > $OUT/pytest_r2n.log 2>&1; echo "pytest rc=$?"; tail -15 $OUT/pytest_r2n.log
timeout 600 python tools/variants_ab.py i8:4096 --flush --reps 40 --rounds 3 --variants "base;MM_STREAMK=4" > $OUT/var_nhalf_r2n.txt 2>&1
timeout 600 python tools/variants_ab.py bf16:4096 --flush --reps 30 --rounds 3 --variants "base;MM_STREAMK=4" >> $OUT/var_nhalf_r2n.txt 2>&1
timeout 600 python tools/variants_ab.py i8:2560 --flush --reps 30 --rounds 3 --variants "base;MM_STREAMK=4" >> $OUT/var_nhalf_r2n.txt 2>&1
timeout 600 python tools/variants_ab.py bf16:2560 --flush --reps 30 --rounds 3 --variants "base;MM_STREAMK=4" >> $OUT/var_nhalf_r2n.txt 2>&1
timeout 600 python tools/variants_ab.py i8:2048x16384x16384 --flush --reps 10 --rounds 2 --variants "base;MM_STREAMK=4" >> $OUT/var_nhalf_r2n.txt 2>&1
timeout 600 python tools/variants_ab.py bf16:3000x5000x4000 --flush --reps 10 --rounds 2 --variants "base;MM_STREAMK=4" >> $OUT/var_nhalf_r2n.txt 2>&1
cat $OUT/var_nhalf_r2n.txt
