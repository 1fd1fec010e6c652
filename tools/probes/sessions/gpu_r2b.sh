# r2b: new bench.py end to end; per-config ncu DRAM traffic; residency A/B old vs new library
set -u
OUT=gpurun_out
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench_r2b.json 2> $OUT/bench_r2b.err; echo "bench rc=$?"
tail -c 600 $OUT/bench_r2b.err
timeout 300 python tools/hazard_ab.py tools/ab/lib_r1.so paper_2408_15384_b200/libmm_b200.so > $OUT/hazard_ab_r2b.txt 2>&1; echo "hazard rc=$?"
for c in f64:256 f64:2000x1500x1750 i8:4096; do
  for L in "" 1; do
    LIB=$L FLUSH=1 timeout 300 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,lts__t_bytes.sum,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed --clock-control none -k 'regex:^(?!distribution|vectorized|elementwise|unrolled|fill).*' -s 2 -c 1 python tools/one_case.py $c 4 2>/dev/null | grep -E "gemm|Kernel|cutlass|dram__|lts__|gpu__time|sm__" | sed "s/^/$c lib=$L /"
  done
done > $OUT/ncu_configs_r2b.txt 2>&1
echo done
