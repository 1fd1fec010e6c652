set -u
OUT=gpurun_out
L=paper_2408_15384_b200
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_hazards.py tests/test_gpu_sharded.py -q -x -k "emulation or emulated or i8 or int8" > $OUT/pytest_emu_r2zz4.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_emu_r2zz4.log
tail -3 $OUT/pytest_emu_r2zz4.log
timeout 900 python tools/probes/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so 2000,1500,1750 4096 8192 16384 32768 > $OUT/ab_emu_epires_r2zz4.txt 2>&1
cat $OUT/ab_emu_epires_r2zz4.txt
timeout 600 python tools/ab_gpu.py $L/libmm_b200_base.so $L/libmm_b200.so --cases i8:4096,i8:8192,bf16:4096,bf16:16384 > $OUT/ab_tc_epires_r2zz4.txt 2>&1; cat $OUT/ab_tc_epires_r2zz4.txt
timeout 300 python tools/probes/emu_once.py 8192 && timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/launches_emu8192_r2zz4.csv python tools/probes/emu_once.py 8192 > /dev/null 2>&1; echo "ncu rc=$?"
