set -u
OUT=gpurun_out
timeout 300 python tools/probes/emu_once.py 16384 > $OUT/emu16k_plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_tc -s 20 -c 1 -o $OUT/prof_emu_gemm_r2zz6 python tools/probes/emu_once.py 16384 > $OUT/ncu_emu_gemm.log 2>&1; echo "ncu1 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:crt_combine -s 1 -c 1 -o $OUT/prof_emu_combine_r2zz6 python tools/probes/emu_once.py 16384 > $OUT/ncu_emu_comb.log 2>&1; echo "ncu2 rc=$?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:residues_a -s 1 -c 1 -o $OUT/prof_emu_res_r2zz6 python tools/probes/emu_once.py 16384 > $OUT/ncu_emu_res.log 2>&1; echo "ncu3 rc=$?"
