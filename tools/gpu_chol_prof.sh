# chol_kernel phase cycles (clock64 stamps) + one ncu --set full capture with source.
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCTM_CHOL_PROF -I paper_2306_08212_b200/csrc \
  tools/bench_iso_kernels.cu -o gpurun_out/bik_prof && timeout 120 gpurun_out/bik_prof 160 > gpurun_out/chol_prof.txt 2>&1
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc \
  tools/bench_iso_kernels.cu -o gpurun_out/bik && timeout 120 gpurun_out/bik 160 > gpurun_out/bik160.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"chol_kernel|trsm_rows" -c 2 \
  -o gpurun_out/chol_full -f gpurun_out/bik 160 > gpurun_out/ncu_chol.log 2>&1
echo "rc=$?" > gpurun_out/rc_chol.txt
