for ks in 1 4; do MM_F64_KS=$ks MM_TRACE=1 timeout 120 python tools/one_case.py f64:256 4 2>&1 | grep "trace f64" | tail -1 | sed "s/^/ks=$ks /"; done
