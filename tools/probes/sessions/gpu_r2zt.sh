set -u
OUT=gpurun_out
L=paper_2408_15384_b200
cat > /tmp/emu_ab.py <<'PY'
import ctypes, statistics, sys, torch
libs = [ctypes.CDLL(p) for p in sys.argv[1:3]]
vp, i64 = ctypes.c_void_p, ctypes.c_int64
hs = []
for lib in libs:
    lib.mm_create.argtypes = [ctypes.c_int, vp, ctypes.c_size_t, ctypes.POINTER(vp)]
    lib.mm_gemm.argtypes = [vp, i64, i64, i64, ctypes.c_int, vp, vp, vp, vp]
    h = vp(); assert lib.mm_create(0, None, 0, ctypes.byref(h)) == 0; hs.append(h)
s = torch.cuda.current_stream().cuda_stream
for N in (2048, 4096, 8192, 16384):
    A = torch.rand(N, N, dtype=torch.float64, device="cuda"); B = torch.rand(N, N, dtype=torch.float64, device="cuda")
    Cs = [torch.empty(N, N, dtype=torch.float64, device="cuda") for _ in libs]
    ts = [[], []]
    for r in range(6):
        for k, (lib, h) in enumerate(zip(libs, hs)):
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record(); assert lib.mm_gemm(h, N, N, N, 3, A.data_ptr(), B.data_ptr(), Cs[k].data_ptr(), s) == 0; e1.record(); e1.synchronize()
            if r: ts[k].append(e0.elapsed_time(e1))
    a, b = statistics.fmean(ts[0]), statistics.fmean(ts[1])
    print(f"F64_EMU {N}^3: A {a:9.3f} ms  B {b:9.3f} ms  B/A speed {a/b:5.3f}  equal={torch.equal(Cs[0], Cs[1])}", flush=True)
PY
python /tmp/emu_ab.py $L/libmm_b200_base.so $L/libmm_b200.so > $OUT/ab_emu_pairs_r2zt.txt 2>&1
cat $OUT/ab_emu_pairs_r2zt.txt
