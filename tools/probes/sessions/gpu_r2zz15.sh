set -u
OUT=gpurun_out
L=paper_2408_15384_b200
{ echo "== MM_WAVE_SYNC=0 on both sides"; MM_WAVE_SYNC=0 timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 4096 8192 16384;
  echo "== MM_WAVE_SYNC=2 (forced) on both sides"; MM_WAVE_SYNC=2 timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 4096 8192 16384; } > $OUT/ab_emu_batched_ws_r2zz15.txt 2>&1
cat $OUT/ab_emu_batched_ws_r2zz15.txt
