# r2o: tail mode sweep over K at 4096 x K x 4096 (256 pair tiles, 34 in the partial round)
set -u
OUT=gpurun_out
: > $OUT/sweep_tail_r2o.txt
for K in 1024 2048 3072 5120 6144 8192; do
  timeout 300 python tools/variants_ab.py i8:4096x${K}x4096 --flush --reps 20 --rounds 2 --variants "MM_STREAMK=0;MM_STREAMK=3;MM_STREAMK=4" >> $OUT/sweep_tail_r2o.txt 2>&1
done
for K in 768 1536 2048 2560 3072 4096; do
  timeout 300 python tools/variants_ab.py bf16:4096x${K}x4096 --flush --reps 20 --rounds 2 --variants "MM_STREAMK=0;MM_STREAMK=3;MM_STREAMK=4" >> $OUT/sweep_tail_r2o.txt 2>&1
done
cat $OUT/sweep_tail_r2o.txt
