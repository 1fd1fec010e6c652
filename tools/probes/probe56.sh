for E in "MM_NT=2 MM_STREAMK=0" "MM_NT=2 MM_STREAMK=1"; do
env $E MM_TRACE=1 FLUSH=1 timeout 120 python tools/one_case.py i8:4096 3 2>&1 | grep "mm trace" | tail -4 | sed "s/^/$E /"
done
L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_NT=2 MM_STREAMK=1 --cases i8:4096,bf16:4096,i8:3072,bf16:3072 --reps 10 2>&1 | tail -4
