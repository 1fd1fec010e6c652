timeout 300 python tools/cublas_shapes.py f64:8192 > /dev/null 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__cycles_active.avg,smsp__inst_executed.sum --clock-control none --csv --log-file gpurun_out/f64_8192_r1z.csv python tools/cublas_shapes.py f64:8192 > /dev/null 2>&1
echo rc=$?
