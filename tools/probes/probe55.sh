for D in 0 2; do
MM_DEBUG=$D MM_TRACE=1 timeout 120 python tools/one_case.py i8:4096 3 2>&1 | grep "mm trace" | grep -v epilogue | tail -3 | sed "s/^/debug=$D /"
done
