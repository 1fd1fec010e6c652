./tools/launch_probe
FLUSH=1 MM_TRACE=1 timeout 120 python tools/one_case.py bf16:256 3 2>&1 | grep "timeline" | tail -1
FLUSH=1 MM_TRACE=1 timeout 120 python tools/one_case.py i8:4096 3 2>&1 | grep "timeline" | tail -1
