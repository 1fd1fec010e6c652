set -u
OUT=gpurun_out
for c in i8:4096 i8:3072; do
  echo "== $c"; MM_B200_LIB=paper_2408_15384_b200/libmm_b200_diag.so MM_TRACE=1 FLUSH=1 timeout 300 python tools/one_case.py $c 3 2>&1 | grep -E "timeline|span|clock|chunk" | tail -4 | cut -c1-1200
done > $OUT/trace_c3_r2zb.txt 2>&1
cat $OUT/trace_c3_r2zb.txt
