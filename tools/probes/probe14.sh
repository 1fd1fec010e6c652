OUT=gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "f64 or fixup or config0 or config1 or config4" > $OUT/pytest_f64st.log 2>&1; echo "pytest rc=$?"; tail -2 $OUT/pytest_f64st.log
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 600 python tools/ab_gpu.py $B $L --cases f64:256,f64:300x200x520,f64:512,f64:1024,f64:2000x1500x1750,f64:8192 --reps 20 2>&1 | tee $OUT/ab_r1t.txt
timeout 600 python tools/ab_gpu.py $L $L --env-b MM_F64_KS=1 --cases f64:256,f64:300x200x520 --reps 20 2>&1 | tee -a $OUT/ab_r1t.txt
