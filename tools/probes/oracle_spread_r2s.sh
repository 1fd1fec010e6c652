set -u
export OMP_NUM_THREADS=16 OMP_PROC_BIND=close OMP_PLACES=cores
echo "standalone worker:"; python bench.py --oracle-worker parallel --threads 16 --config C4
echo "oracle_baseline() from a plain python:"; python -c "import bench, json; r=bench.oracle_baseline(('parallel',)); print(json.dumps(r['parallel']['C4']))"
echo "from a process holding a CUDA context + pinned memory:"; python -c "
import torch, bench, json, numpy as np
x = torch.empty(2<<30, dtype=torch.uint8).pin_memory(); y = torch.ones(1, device='cuda'); torch.cuda.synchronize()
r=bench.oracle_baseline(('parallel',)); print(json.dumps(r['parallel']['C4']))"
echo "reference arm:"; python bench.py --impl reference --steps 3 --warmup 1 | head -c 250; echo
nproc; cat /sys/kernel/mm/transparent_hugepage/enabled; numactl -H 2>/dev/null | head -3; free -g | head -2
