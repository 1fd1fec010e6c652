timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 300 python tools/overhead_probe.py --cases f64:256,bf16:128,i8:4096 2>&1
