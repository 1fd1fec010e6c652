L=paper_2408_15384_b200/libmm_b200.so
C=i8:4096,bf16:4096,i8:3072,i8:6144,bf16:6144
for E in "MM_NT=1" "MM_NT=1 MM_STREAMK=2" "MM_NT=1 MM_STREAMK=1" "MM_NT=1 MM_KA=1"; do
 echo "== B: $E"; timeout 600 python tools/ab_gpu.py $L $L --env-b $E --cases $C --reps 10 2>&1 | tail -5
done
