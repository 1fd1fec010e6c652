set -u
OUT=gpurun_out; mkdir -p $OUT
timeout 300 python tools/cublas_shapes.py > /dev/null 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,sm__cycles_elapsed.avg.per_second,sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_requests_srcunit_tex_op_read.sum --clock-control none --csv --log-file $OUT/cublas_shapes_r1h.csv python tools/cublas_shapes.py > $OUT/ncu_cublas_shapes_r1h.log 2>&1
echo "rc=$?"
