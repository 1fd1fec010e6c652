set -u
OUT=gpurun_out
timeout 300 python tools/probes/c3_once.py > $OUT/c3_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none -s 4 -c 2 -o $OUT/prof_c3_r2zz24 python tools/probes/c3_once.py > $OUT/ncu_c3.log 2>&1; echo "ncu rc=$?"
