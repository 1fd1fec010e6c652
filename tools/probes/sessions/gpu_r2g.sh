# r2g: non-persistent (one tile per cluster) vs persistent: C3 and C4 vs cuBLAS; ncu L2 sectors for C3
set -u
OUT=gpurun_out
timeout 600 python tools/variants_ab.py i8:4096 --flush --reps 40 --rounds 3 --variants "base;MM_ONE_TILE=1;MM_ONE_TILE=1,MM_NT=2;MM_ONE_TILE=1,MM_KA=1" > $OUT/var_c3_r2g.txt 2>&1; cat $OUT/var_c3_r2g.txt
timeout 900 python tools/variants_ab.py bf16:16384 --window-s 2 --rounds 2 --variants "base;MM_ONE_TILE=1;MM_ONE_TILE=1,MM_NT=1" > $OUT/var_c4_r2g.txt 2>&1; cat $OUT/var_c4_r2g.txt
MM_ONE_TILE=1 FLUSH=1 timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_ltcfabric.sum,sm__ops_path_tensor_op_utcimma_src_int8_sparsity_off.avg.pct_of_peak_sustained_elapsed --clock-control none -k regex:gemm_tc -s 2 -c 1 python tools/one_case.py i8:4096 4 2>/dev/null | grep -E "gemm|lts|gpu__|sm__" > $OUT/ncu_c3_onetile_r2g.txt; cat $OUT/ncu_c3_onetile_r2g.txt
