for d in 1 17; do MM_DEBUG=$d MM_NT=2 MM_TRACE=1 timeout 120 python tools/one_case.py i8:4096 4 2>&1 | grep "timeline\|clock" | tail -2 | sed "s/^/debug=$d /"; done
for d in 1 17; do MM_DEBUG=$d MM_NT=2 MM_TRACE=1 timeout 120 python tools/one_case.py bf16:8192 4 2>&1 | grep "timeline\|clock" | tail -2 | sed "s/^/debug=$d /" | cut -c1-250; done
