set -u
OUT=gpurun_out
L=paper_2408_15384_b200
timeout 1500 python -m pytest tests/test_gpu_parity.py -q -x -k "emulation or emulated" > $OUT/pytest_emu_r2zv.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_emu_r2zv.log
tail -3 $OUT/pytest_emu_r2zv.log
timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 2000,1500,1750 2048 4096 8192 16384 32768 > $OUT/ab_emu_crt_r2zv.txt 2>&1
cat $OUT/ab_emu_crt_r2zv.txt
