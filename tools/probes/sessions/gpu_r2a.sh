set -u
OUT=gpurun_out
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_r2a.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke_r2a.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_r2a.log
timeout 900 python -m pytest tests/test_gpu_hazards.py tests/test_gpu_ipc.py tests/test_gpu_sharded.py tests/test_dist_nccl.py -q -rs > $OUT/pytest_new_r2a.log 2>&1; echo "rc=$?" >> $OUT/pytest_new_r2a.log
timeout 1500 python -m pytest tests -m gpu -q -rs --deselect tests/test_dist_nccl.py > $OUT/pytest_gpu_r2a.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_r2a.log
tail -3 $OUT/smoke_r2a.log $OUT/pytest_new_r2a.log $OUT/pytest_gpu_r2a.log
