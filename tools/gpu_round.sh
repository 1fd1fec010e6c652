#!/bin/bash
# One GPU session: smoke, the whole GPU suite, bench, then (only if the identical plain command
# exited 0) an ncu launch list and a full capture of the top kernel.
#   tools/gpu_round.sh [tag] [what]    what: all | tests | bench | ncu
set -u
TAG=${1:-r2}
WHAT=${2:-all}
OUT=gpurun_out
mkdir -p $OUT
nvidia-smi --query-gpu=name,driver_version,clocks.sm,clocks.max.sm,power.draw --format=csv > $OUT/gpu_$TAG.txt 2>&1
lscpu | grep -E "Model name|^CPU\(s\)|Socket|Core" >> $OUT/gpu_$TAG.txt 2>&1
if [[ $WHAT == all || $WHAT == tests ]]; then
  timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $OUT/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke_$TAG.log
  timeout 2400 python -m pytest tests -m gpu -q -rs > $OUT/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu_$TAG.log
  tail -5 $OUT/pytest_gpu_$TAG.log
fi
if [[ $WHAT == all || $WHAT == bench ]]; then
  timeout 1200 python bench.py --steps 20 --warmup 5 > $OUT/bench_$TAG.json 2> $OUT/bench_$TAG.err; echo "bench rc=$?"
  timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $OUT/bench_ref_$TAG.json 2> $OUT/bench_ref_$TAG.err; echo "ref rc=$?"
fi
if [[ $WHAT == all || $WHAT == ncu ]]; then
  CMD="python bench.py --steps 10 --warmup 3 --no-per-config --no-cpu-baseline --no-protocol --no-sustained --no-k6"
  timeout 600 $CMD > $OUT/ncu_plain_$TAG.log 2>&1 && \
  timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv \
      --log-file $OUT/launches_$TAG.csv $CMD > $OUT/ncu_launch_$TAG.log 2>&1 && \
  timeout 1200 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 3 -c 1 \
      -o $OUT/prof_bf16_$TAG $CMD > $OUT/ncu_full_$TAG.log 2>&1
  echo "ncu rc=$?"
fi
