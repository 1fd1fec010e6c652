for d in 0 1; do for s in i8:4096 bf16:4096; do MM_DEBUG=$d MM_NT=1 MM_TRACE=1 timeout 120 python tools/one_case.py $s 4 2>&1 | grep "timeline\|clock" | tail -2 | sed "s/^/debug=$d $s /"; done; done
