# r2k: C3 timelines, whole-tile tail vs reduce-add K halves (diag build)
set -u
OUT=gpurun_out
for V in "" "MM_STREAMK=3" "MM_STREAMK=2"; do
  echo "== $V"; env $V MM_B200_LIB=paper_2408_15384_b200/libmm_b200_diag.so MM_TRACE=1 FLUSH=1 timeout 300 python tools/one_case.py i8:4096 3 2>&1 | tail -4 | cut -c1-900
done > $OUT/trace_c3_tails_r2k.txt 2>&1; cat $OUT/trace_c3_tails_r2k.txt
