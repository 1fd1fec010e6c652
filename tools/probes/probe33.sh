for ks in 1 2 4 8 44; do MM_F64_KS=$ks MM_TRACE=1 timeout 120 python tools/one_case.py f64:256 4 2>&1 | grep "trace f64" | tail -1 | sed "s/^/ks=$ks /"; done
L=paper_2408_15384_b200/libmm_b200.so
for ks in 2 8 44; do timeout 600 python tools/ab_gpu.py $L $L --env-a MM_F64_KS=4 --env-b MM_F64_KS=$ks --cases f64:256 --reps 20 2>&1 | sed "s/^/A=ks4 B=ks$ks /"; done
