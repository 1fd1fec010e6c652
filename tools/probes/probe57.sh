for c in f64:8192 f64:16384; do for L in "" 1; do
LIB=$L timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,sm__cycles_elapsed.avg.per_second --clock-control none --csv -k 'regex:^(?!distribution|vectorized|elementwise|unrolled).*' -s 1 -c 1 python tools/one_case.py $c 3 2>/dev/null | grep -E "gpu__time|dram__|lts__|per_second" | awk -F'","' '{print substr($5,1,50)" | "$(NF-2)" "$(NF-1)" "$NF}' | sed "s/^/$c lib=$L /"
done; done
