for c in bf16:2048 i8:3072; do
MM_TRACE=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | tail -4
MM_TRACE=1 MM_DEBUG=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | tail -4 | sed 's/^/noload /'
done
