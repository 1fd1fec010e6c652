set -u
OUT=gpurun_out
python tools/one_case.py f64:8192 2 > /dev/null 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_f64 -s 1 -c 1 -o $OUT/prof_f64_ours_r2zp python tools/one_case.py f64:8192 2 > $OUT/ncu_f64_ours_r2zp.log 2>&1
LIB=1 timeout 900 ncu --set full --clock-control none -k regex:gemm -s 1 -c 1 -o $OUT/prof_f64_lib_r2zp python tools/one_case.py f64:8192 2 > $OUT/ncu_f64_lib_r2zp.log 2>&1
ls -la $OUT/*.ncu-rep
