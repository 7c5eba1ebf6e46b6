nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -DCTM_CHOL_PROF -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o gpurun_out/bik_prof && (timeout 60 gpurun_out/bik_prof 160; timeout 60 gpurun_out/bik_prof 100) > gpurun_out/chol_prof.txt 2>&1
SWEEP=c4,c5 BIK_SIZES="128 160" bash tools/gpu_iso_quick.sh
