# r2j: FP64 K-split clusters for small problems (C1) + k-phase pacing for C4
set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -q -x -k "f64 or fuzz or brute or hand or identity" > $OUT/pytest_r2j.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_r2j.log
MM_PACE=8 timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "bf16 and (16384 or config3 or row_block)" > $OUT/pytest_r2j_pace.log 2>&1; echo "pace pytest rc=$?"; tail -1 $OUT/pytest_r2j_pace.log
timeout 600 python tools/variants_ab.py f64:256 --graph --reps 20 --rounds 3 --variants "base;MM_F64_CK=1" > $OUT/var_c1_r2j.txt 2>&1; cat $OUT/var_c1_r2j.txt
timeout 600 python tools/variants_ab.py f64:256 --flush --reps 40 --rounds 3 --variants "base;MM_F64_CK=1" >> $OUT/var_c1_r2j.txt 2>&1; tail -3 $OUT/var_c1_r2j.txt
timeout 600 python tools/variants_ab.py f64:128x512x200 --graph --reps 20 --rounds 2 --variants "base;MM_F64_CK=1" >> $OUT/var_c1_r2j.txt 2>&1; tail -3 $OUT/var_c1_r2j.txt
timeout 1200 python tools/variants_ab.py bf16:16384 --window-s 2 --rounds 2 --variants "base;MM_PACE=4;MM_PACE=8;MM_PACE=16;MM_PACE=32" > $OUT/var_c4_pace_r2j.txt 2>&1; cat $OUT/var_c4_pace_r2j.txt
for V in "" "MM_PACE=8" "MM_PACE=16"; do
  env $V timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,dram__bytes_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 python tools/one_case.py bf16:16384 3 2>/dev/null | grep -E "lts|gpu__|dram|sm__" | sed "s/^/[$V] /"
done > $OUT/ncu_c4_pace_r2j.txt 2>&1; cat $OUT/ncu_c4_pace_r2j.txt
