# r2h: C3 tail-split variants; L2 sector reads vs wave alignment
set -u
OUT=gpurun_out
timeout 600 python tools/variants_ab.py i8:4096 --flush --reps 40 --rounds 3 --variants "base;MM_STREAMK=1;MM_STREAMK=2;MM_STREAMK=3;MM_GROUP_M=16;MM_GROUP_M=1" > $OUT/var_c3_r2h.txt 2>&1; cat $OUT/var_c3_r2h.txt
for V in "" "MM_WAVE_SYNC=2" "MM_STREAMK=2" "MM_GROUP_M=16"; do
  env $V FLUSH=1 timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_ltcfabric.sum,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tc -s 2 -c 1 python tools/one_case.py i8:4096 4 2>/dev/null | grep -E "lts|gpu__|sm__" | sed "s/^/[$V] /"
done > $OUT/ncu_c3_variants_r2h.txt 2>&1; cat $OUT/ncu_c3_variants_r2h.txt
