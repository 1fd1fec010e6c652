set -u
OUT=gpurun_out
L=paper_2408_15384_b200
{ echo "== A = new (small-product batching), B = base"; timeout 900 python tools/probes/emu_ab.py $L/libmm_b200.so $L/libmm_b200_base.so 4096 8192 16384 32768;
  echo "== A = base, B = new"; timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 4096 8192 16384 32768; } > $OUT/ab_emu_order_r2zz18.txt 2>&1; cat $OUT/ab_emu_order_r2zz18.txt
