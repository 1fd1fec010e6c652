set -u
OUT=gpurun_out
for I in 0 0.5 2 0 0.5 2; do
  timeout 600 python bench.py --steps 20 --warmup 5 --idle-s $I --no-per-config --no-cpu-baseline --no-protocol --no-sustained > $OUT/b.json 2>/dev/null
  python -c "import json; d=json.load(open('$OUT/b.json')); print('idle', $I, d['value'], d['ms_per_step'], d['clocks'])"
done > $OUT/idle_r2w.txt 2>&1; cat $OUT/idle_r2w.txt
