for G in 16 8; do for H in 0 1 3; do
MM_GROUP_M=$G MM_L2_HINT=$H timeout 600 ncu --metrics dram__bytes_read.sum,gpu__time_duration.sum,sm__cycles_elapsed.avg.per_second --clock-control none -k regex:gemm_tc -s 1 -c 1 python tools/one_case.py bf16:16384 2 2>/dev/null | grep -E "dram__|gpu__|per_second" | awk '{print $1, $(NF-1), $NF}' | tr '\n' ' ' | sed "s/^/group=$G hint=$H /"; echo
done; done
