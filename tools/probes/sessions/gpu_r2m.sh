# r2m: wave-barrier / pacing poll back-off (hot L2 slice hypothesis)
set -u
OUT=gpurun_out
timeout 1800 python tools/variants_ab.py bf16:16384 --window-s 2 --rounds 2 --variants "base;MM_POLL_NS=256;MM_POLL_NS=1024;MM_PACE=16,MM_POLL_NS=512;MM_PACE=32,MM_POLL_NS=512;MM_PACE=8,MM_POLL_NS=1024;MM_PACE=64,MM_POLL_NS=512" > $OUT/var_c4_poll_r2m.txt 2>&1; cat $OUT/var_c4_poll_r2m.txt
for V in "" "MM_POLL_NS=1024" "MM_PACE=16 MM_POLL_NS=512" "MM_PACE=32 MM_POLL_NS=512"; do
  env $V timeout 300 ncu --metrics gpu__time_duration.sum,lts__t_sectors_srcunit_tex_op_read.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 2 -c 1 python tools/one_case.py bf16:16384 3 2>/dev/null | grep -E "lts|gpu__|sm__" | sed "s/^/[$V] /"
done > $OUT/ncu_c4_poll_r2m.txt 2>&1; cat $OUT/ncu_c4_poll_r2m.txt
