B=paper_2408_15384_b200/libmm_b200_base.so; L=paper_2408_15384_b200/libmm_b200.so
nvidia-smi --query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_event_reasons.active --format=csv -lms 500 > gpurun_out/clk_r1p.csv 2>&1 &
SMI=$!
timeout 900 python tools/ab_gpu.py $B $L --cases i8:4096,bf16:4096,i8:8192,bf16:8192 --reps 10 2>&1 | tee gpurun_out/ab_r1p.txt
timeout 900 python tools/ab_gpu.py $L $L --env-a MM_NT=1 --env-b MM_NT=2 --cases i8:4096,bf16:4096 --reps 10 2>&1 | tee -a gpurun_out/ab_r1p.txt
kill $SMI
