set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "mc2" > $OUT/pytest_mc2.log 2>&1; echo "pytest rc=$?"; tail -5 $OUT/pytest_mc2.log
L=paper_2408_15384_b200/libmm_b200.so
cp $L /tmp/libB.so
timeout 600 python tools/ab_gpu.py $L /tmp/libB.so --env-b MM_MC=2 --cases bf16:4096,bf16:8192,bf16:16384,i8:4096,i8:8192,bf16:2048 --reps 10 2>&1 | tee $OUT/ab_mc2.txt
timeout 600 python tools/ab_gpu.py $L /tmp/libB.so --env-a MM_NT=1 --env-b MM_MC=2 MM_NT=1 --cases bf16:8192,bf16:16384,i8:8192 --reps 10 2>&1 | tee $OUT/ab_mc2_nt1.txt
