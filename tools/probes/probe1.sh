set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python tools/overhead_probe.py > $OUT/overhead_r1g.txt 2>&1; echo "probe rc=$?"
cat $OUT/overhead_r1g.txt
for c in i8:4096 f64:256 f64:2000x1500x1750; do
  tag=$(echo $c | tr ':x' '__')
  timeout 300 python tools/one_case.py $c 5 > /dev/null 2>&1 && \
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:gemm_ -s 3 -c 1 -o $OUT/prof_${tag}_r1g python tools/one_case.py $c 5 > $OUT/ncu_${tag}_r1g.log 2>&1
  echo "ncu $c rc=$?"
done
