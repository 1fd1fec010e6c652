nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/occ tools/occ_probe.cu && /tmp/occ | tee gpurun_out/occ_r1.txt
