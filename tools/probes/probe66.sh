for c in i8:4096 i8:2560 bf16:4096; do for M in 0 3; do
FLUSH=1 MM_STREAMK=$M MM_TRACE=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | grep -v "epilogue cycles" | tail -3 | sed "s/^/$c sk=$M /"
done; done
