timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "tc or wide or mc2 or tiny or handworked or fixup or config2 or epilogue" 2>&1 | tail -2
for d in 1 0; do for nt in 1 2; do MM_DEBUG=$d MM_NT=$nt MM_TRACE=1 timeout 120 python tools/one_case.py i8:4096 4 2>&1 | grep "timeline\|clock" | tail -2 | sed "s/^/debug=$d nt=$nt /"; done; done
