set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
{
for E in MM_NT=1 MM_GROUP_M=8 MM_GROUP_M=4 MM_WAVE_SYNC=2; do
echo "== B: $E"
timeout 600 python tools/ab_gpu.py $L $L --env-b $E --reps 20 --cases i8:4096x4096x8192,i8:8192x4096x4096,i8:6144,bf16:4096x4096x8192
done
} > $OUT/ab_r2zi.txt 2>&1
cat $OUT/ab_r2zi.txt
MM_B200_LIB=paper_2408_15384_b200/libmm_b200_diag.so MM_TRACE=1 FLUSH=1 timeout 300 python tools/one_case.py i8:4096x4096x8192 3 2>&1 | grep -E "timeline|span|clock|chunk" | tail -4 | cut -c1-1500
