set -u
OUT=gpurun_out
L=paper_2408_15384_b200
timeout 900 python tools/ab_gpu.py $L/libmm_b200_base.so $L/libmm_b200.so --cases f64:4096,f64:8192,f64:2000x1500x1750,f64:16384,i8:4096,bf16:8192 > $OUT/ab_f64_nospill_r2zz9.txt 2>&1; cat $OUT/ab_f64_nospill_r2zz9.txt
timeout 600 python -m pytest tests/test_gpu_hazards.py -q -x -k clock > $OUT/pytest_clk.log 2>&1; tail -1 $OUT/pytest_clk.log
