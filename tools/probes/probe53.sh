FLUSH=1 MM_TRACE=1 timeout 120 python tools/one_case.py bf16:256 3 2>&1 | grep "mm trace" | grep -v epilogue | tail -3
mkdir -p gpurun_out
for L in "" 1; do
LIB=$L FLUSH=1 timeout 300 ncu --metrics gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none --csv python tools/one_case.py bf16:256 4 2>/dev/null | grep -v fill | grep -E "gpu__time|per_second" | tail -4
done
for L in "" 1; do
LIB=$L FLUSH=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv python tools/one_case.py i8:4096 4 2>/dev/null | grep -v fill | grep -E "gpu__time" | tail -2
done
