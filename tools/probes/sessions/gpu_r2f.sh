# r2f: deep profiles of C3 (INT8 4096^3) and C4 (BF16 16384^3): ours vs cuBLAS, ncu --set full; C3 timeline (diag build)
set -u
OUT=gpurun_out
for LIBV in "" 1; do
  LIB=$LIBV FLUSH=1 timeout 900 ncu --set full --clock-control none --import-source on -k 'regex:^(?!distribution|vectorized|elementwise|unrolled|fill).*' -s 2 -c 1 -f -o $OUT/prof_c3_lib${LIBV:-0}_r2f python tools/one_case.py i8:4096 4 > $OUT/ncu_c3_lib${LIBV:-0}_r2f.log 2>&1; echo "c3 lib=$LIBV rc=$?"
done
for V in "base" "MM_MC=2" "LIB=1"; do
  if [ "$V" = "base" ]; then E=""; else E="$V"; fi
  env $E timeout 1200 ncu --set full --clock-control none -k 'regex:^(?!distribution|vectorized|elementwise|unrolled|fill).*' -s 2 -c 1 -f -o $OUT/prof_c4_${V//=/_}_r2f python tools/one_case.py bf16:16384 3 > $OUT/ncu_c4_${V//=/_}_r2f.log 2>&1; echo "c4 $V rc=$?"
done
MM_B200_LIB=paper_2408_15384_b200/libmm_b200_diag.so MM_TRACE=1 FLUSH=1 timeout 300 python tools/one_case.py i8:4096 4 > $OUT/trace_c3_r2f.txt 2>&1; echo "trace rc=$?"; tail -4 $OUT/trace_c3_r2f.txt
ls -la $OUT/*.ncu-rep
