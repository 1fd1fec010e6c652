M=gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,launch__registers_per_thread,launch__grid_size,launch__block_size,sm__cycles_active.avg,sm__cycles_elapsed.avg
for c in i8:4096 f64:2000x1500x1750 f64:256; do for L in "" 1; do
echo "== $c lib=$L"
LIB=$L FLUSH=1 timeout 600 ncu --metrics $M --clock-control none -k 'regex:^(?!distribution|vectorized|elementwise|unrolled).*' -s 2 -c 1 python tools/one_case.py $c 4 2>/dev/null | grep -E "^  [a-zA-Z]|gpu__|sm__|dram__|lts__|launch__" | sed 's/  */ /g' | cut -c1-150
done; done
