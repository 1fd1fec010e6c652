set -u
OUT=gpurun_out
timeout 1800 python -m pytest tests/test_gpu_sharded.py tests/test_gpu_shim_multirank.py tests/test_gpu_hazards.py -q -x -k "not full" > $OUT/pytest_emu_shard_r2zz.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_emu_shard_r2zz.log
tail -3 $OUT/pytest_emu_shard_r2zz.log
