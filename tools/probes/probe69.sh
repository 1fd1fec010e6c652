for D in 0 1 4 5; do
MM_DEBUG=$D FLUSH=1 timeout 600 ncu --metrics lts__t_bytes.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_write.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_write.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_atom.sum,dram__bytes_read.sum,gpu__time_duration.sum --clock-control none -k regex:gemm_tc -s 2 -c 1 python tools/one_case.py i8:4096 4 2>/dev/null | grep -E "lts__|dram__|gpu__" | sed "s/^/debug=$D /"
done
