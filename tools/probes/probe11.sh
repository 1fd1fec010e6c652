OUT=gpurun_out
for nt in 1 2; do MM_TRACE=1 MM_NT=$nt timeout 120 python tools/one_case.py i8:4096 3 2>&1 | grep "mm trace" | tail -1; done | tee $OUT/trace_i8_r1q.txt
for c in i8:4096 f64:256; do
  tag=$(echo $c | tr ':x' '__')
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -s 3 -c 1 -o $OUT/prof_${tag}_r1q python tools/one_case.py $c 5 > $OUT/ncu_${tag}_r1q.log 2>&1
  echo "ncu $c rc=$?"
done
