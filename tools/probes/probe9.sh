python tools/dbg_f64.py 128 1 60 | tail -3
python tools/dbg_f64.py 64 1 30 | tail -1
python tools/dbg_f64.py 32 1 30 | tail -1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_fix3.log 2>&1; echo "pytest rc=$?"; tail -4 gpurun_out/pytest_gpu_fix3.log
B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
timeout 900 python tools/ab_gpu.py $B $L --cases f64:256,f64:2000x1500x1750,f64:8192,bf16:4096,bf16:8192,bf16:16384,i8:4096,i8:8192 --reps 10 2>&1 | tee gpurun_out/ab_r1o.txt
