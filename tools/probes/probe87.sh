for H in 0 4; do
MM_L2_HINT=$H timeout 600 ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 1 -c 1 python tools/one_case.py bf16:16384 2 2>/dev/null | grep -E "dram__|gpu__|per_second" | awk '{print $1, $(NF-1), $NF}' | tr '\n' ' ' | sed "s/^/hint=$H /"; echo
done
L=paper_2408_15384_b200/libmm_b200.so
timeout 300 python tools/ab_gpu.py $L $L --env-b MM_L2_HINT=4 --cases i8:4096,bf16:8192 --reps 10 2>&1 | tail -2
