for c in bf16:2048 i8:4096; do
FLUSH=1 MM_TRACE=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | grep -v epilogue | tail -3
FLUSH=1 MM_TRACE=1 MM_NO_PDL=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | grep -v epilogue | tail -3 | sed 's/^/nopdl /'
done
