python tools/dbg_f64.py 128 1 60
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_fix2.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_fix2.log
