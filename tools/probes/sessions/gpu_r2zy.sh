set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
C=i8:4096,i8:3072,i8:6144,i8:8192,bf16:4096,bf16:8192
{ echo "== B: MM_MC=2 MM_NT=1 (4-CTA clusters, 512x256 tiles, KA=2)"; timeout 600 python tools/ab_gpu.py $L $L --env-b MM_MC=2 MM_NT=1 --cases $C;
  echo "== B: MM_MC=2 MM_NT=2 (4-CTA clusters, 512x512 tiles)"; timeout 600 python tools/ab_gpu.py $L $L --env-b MM_MC=2 MM_NT=2 --cases $C; } > $OUT/ab_mc2_r2zy.txt 2>&1
cat $OUT/ab_mc2_r2zy.txt
