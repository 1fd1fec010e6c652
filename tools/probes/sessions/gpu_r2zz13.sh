set -u
OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "host_operand" > $OUT/pytest_host_emu.log 2>&1; tail -1 $OUT/pytest_host_emu.log
timeout 1200 python tools/probes/f64_emu_probe.py 512 1024 2048 3072 4096 6144 8192 12288 16384 32768 > $OUT/f64_emu_sweep_r2zz13.txt 2>&1; cat $OUT/f64_emu_sweep_r2zz13.txt
