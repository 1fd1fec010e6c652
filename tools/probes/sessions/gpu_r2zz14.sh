set -u
OUT=gpurun_out
L=paper_2408_15384_b200
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hazards.py tests/test_gpu_sharded.py tests/test_gpu_fuzz.py tests/test_gpu_shim_multirank.py -q -x -k "emulation or emulated or emu or host_operand" > $OUT/pytest_batch_r2zz14.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_batch_r2zz14.log
tail -3 $OUT/pytest_batch_r2zz14.log
timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 2000,1500,1750 1024 2048 4096 8192 16384 32768 > $OUT/ab_emu_batched_r2zz14.txt 2>&1
cat $OUT/ab_emu_batched_r2zz14.txt
