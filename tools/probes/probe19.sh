L=paper_2408_15384_b200/libmm_b200.so
OUT=gpurun_out
for envb in "MM_WAVE_SYNC=2" "MM_GROUP_M=4" "MM_GROUP_M=8" "MM_NT=1 MM_STREAMK=2" "MM_NT=1 MM_GROUP_M=4"; do
  echo "== B: $envb"
  timeout 300 python tools/ab_gpu.py $L $L --env-b $envb --cases i8:4096,bf16:4096 --reps 12 2>&1
done | tee $OUT/ab_c3_r1x.txt
