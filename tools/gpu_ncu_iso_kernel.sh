# ncu --set full (with source) of one launch of an isometry-solver kernel from the microbenchmark.
#   KREGEX=jacobi_cluster N=160 bash tools/gpu_ncu_iso_kernel.sh
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc \
  tools/bench_iso_kernels.cu -o gpurun_out/bik && timeout 120 gpurun_out/bik ${N:-160} > gpurun_out/bik_n.txt 2>&1 && \
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"${KREGEX}" --launch-skip ${SKIP:-0} -c ${COUNT:-1} \
  -o gpurun_out/iso_kernel_full -f gpurun_out/bik ${N:-160} > gpurun_out/ncu_iso_kernel.log 2>&1
echo "rc=$?" > gpurun_out/rc_ncuk.txt
