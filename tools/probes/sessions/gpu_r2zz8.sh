set -u
OUT=gpurun_out
L=paper_2408_15384_b200/libmm_b200.so
C=i8:4096,i8:3072,i8:6144,bf16:4096,i8:8192
{ for E in 8 264 520 2056; do echo "== B: MM_EXP=$E (column-group pacing, P = $(( (E >> 8) ? (E >> 8) : 4 )))"; timeout 600 python tools/ab_gpu.py $L $L --env-b MM_EXP=$E --cases $C; done; } > $OUT/ab_gpace_r2zz8.txt 2>&1
cat $OUT/ab_gpace_r2zz8.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "int8 and not full" > $OUT/pytest_gp.log 2>&1; tail -1 $OUT/pytest_gp.log
