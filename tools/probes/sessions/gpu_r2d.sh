# r2d: FP64 32-bit smem addressing A/B; C4 sustained and C3 schedule variants vs cuBLAS; ncu FP64 C5
set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
timeout 300 python -m pytest tests/test_gpu_parity.py -q -x -k "f64" > $OUT/pytest_r2d.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_r2d.log; tail -2 $OUT/pytest_r2d.log
timeout 900 python tools/ab_gpu.py tools/ab/lib_head.so $L --cases f64:2000x1500x1750,f64:4096,f64:8192,f64:16384,f64:256 --reps 12 > $OUT/ab_f64lds_r2d.txt 2>&1
timeout 900 python tools/ab_gpu.py tools/ab/lib_head.so $L --cases f64:32768 --reps 3 >> $OUT/ab_f64lds_r2d.txt 2>&1
cat $OUT/ab_f64lds_r2d.txt
timeout 1200 python tools/variants_ab.py bf16:16384 --window-s 2 --rounds 2 --variants "base;MM_NT=1;MM_MC=2;MM_GROUP_M=8;MM_GROUP_M=32;MM_WAVE_SYNC=0;MM_L2_HINT=1" > $OUT/var_c4_r2d.txt 2>&1; cat $OUT/var_c4_r2d.txt
timeout 900 python tools/variants_ab.py i8:4096 --flush --reps 40 --rounds 3 --variants "base;MM_NT=2;MM_MC=2;MM_GROUP_M=2;MM_GROUP_M=8;MM_KA=1;MM_STREAMK=3;MM_WAVE_SYNC=2;MM_NT=2,MM_MC=2" > $OUT/var_c3_r2d.txt 2>&1; cat $OUT/var_c3_r2d.txt
for LIBV in "" 1; do
  LIB=$LIBV timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_elapsed.avg.per_second --clock-control none -k 'regex:^(?!distribution|vectorized|elementwise|unrolled|fill).*' -s 1 -c 1 python tools/one_case.py f64:32768 2 2>/dev/null | grep -E "gemm|Kernel|dram__|lts__|gpu__time|sm__" | sed "s/^/lib=$LIBV /"
done > $OUT/ncu_f64_c5_r2d.txt 2>&1; cat $OUT/ncu_f64_c5_r2d.txt
