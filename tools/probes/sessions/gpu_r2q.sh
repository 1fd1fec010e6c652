set -u
OUT=gpurun_out
for c in bf16:2560 bf16:4096 i8:4096; do
  echo "== $c"; MM_B200_LIB=paper_2408_15384_b200/libmm_b200_diag.so MM_TRACE=1 FLUSH=1 timeout 300 python tools/one_case.py $c 3 2>&1 | grep -E "timeline|span|clock" | tail -3 | cut -c1-1000
  LIB=1 FLUSH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k 'regex:^(?!distribution|vectorized|elementwise|unrolled|fill).*' -s 2 -c 1 python tools/one_case.py $c 4 2>/dev/null | grep -E "^  [a-z_0-9]|gpu__time" | head -3
done > $OUT/trace_mid_r2q.txt 2>&1; cat $OUT/trace_mid_r2q.txt
