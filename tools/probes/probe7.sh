python tools/dbg_f64.py 128 1 40
python tools/dbg_f64.py 128 0 40
python tools/dbg_f64.py 64 1 40
python tools/dbg_f64.py 128 1 40 2000 1500 1750
