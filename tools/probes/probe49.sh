L=paper_2408_15384_b200/libmm_b200.so
C=i8:4096,bf16:4096,i8:3072,bf16:3072,i8:6144,i8:8192
for E in "MM_MC=2 MM_NT=1" "MM_MC=2"; do
 echo "== B: $E"; timeout 600 python tools/ab_gpu.py $L $L --env-b $E --cases $C --reps 10 2>&1 | tail -6
done
for c in i8:4096; do
MM_TRACE=1 MM_MC=2 MM_NT=1 timeout 120 python tools/one_case.py $c 3 2>&1 | grep "mm trace" | tail -4
done
