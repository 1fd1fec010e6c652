for D in 0 16; do for c in i8:4096 bf16:256; do
MM_DEBUG=$D FLUSH=1 MM_TRACE=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "timeline" | tail -1 | cut -c1-200 | sed "s/^/dbg=$D $c /"
done; done
