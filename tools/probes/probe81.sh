for F in "" 1; do
FLUSH=$F MM_TRACE=1 timeout 120 python tools/one_case.py f64:256 4 2>&1 | grep "mm trace f64" | tail -1 | sed "s/^/flush=$F /"
done
