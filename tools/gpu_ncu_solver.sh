# ncu --set full captures of the isometry solver's serial kernels (microbenchmark at l = 160 / n = 128)
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc \
  tools/bench_iso_kernels.cu -o gpurun_out/bik && timeout 60 gpurun_out/bik 160 > gpurun_out/bik160.txt 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:chol_kernel -c 1 -o gpurun_out/solver_chol -f gpurun_out/bik 160 > gpurun_out/ncu_s1.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:trsm_rows -c 1 -o gpurun_out/solver_trsm -f gpurun_out/bik 160 > gpurun_out/ncu_s2.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:jacobi_cluster --launch-skip 4 -c 1 -o gpurun_out/solver_jacobi -f gpurun_out/bik 128 > gpurun_out/ncu_s3.log 2>&1
echo done > gpurun_out/rc_ncus.txt
