for D in 0 1; do for c in i8:4096 bf16:4096; do
MM_TRACE=1 MM_DEBUG=$D timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | tail -4 | sed "s/^/debug=$D $c /"
done; done
