mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc tools/bench_iso_kernels.cu -o gpurun_out/bik && (for n in 64 100 160; do timeout 60 gpurun_out/bik $n; done) 2>&1 | grep "trsm\|chol" > gpurun_out/trsm_warm.txt
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:trsm_rows -c 3 --csv gpurun_out/bik 160 > gpurun_out/trsm_cold.csv; timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:chol_kernel -c 3 --csv gpurun_out/bik 160 > gpurun_out/chol_cold.csv 2>&1 2>&1
SWEEP=c3,c4,c5 bash tools/gpu_full_check.sh
