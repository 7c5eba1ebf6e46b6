# C5 isometry-solver check: kernel microbench (l = 160, 232, 288), ISO parity tests,
# (D, chi) sweep incl. C5 with the ISO solver.
mkdir -p gpurun_out
rm -f gpurun_out/rc_c5.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc \
  tools/bench_iso_kernels.cu -o gpurun_out/bench_iso_kernels && \
  for n in 160 232 288; do timeout 120 gpurun_out/bench_iso_kernels $n; done > gpurun_out/bench_iso_kernels_c5.txt 2>&1
echo "microbench rc=$?" >> gpurun_out/rc_c5.txt
timeout 1500 python -m pytest tests -m gpu -q -rA -x -k "iso" --durations=15 > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_c5.txt
timeout 900 python tools/sweep.py --configs c4,c5,c5_256 --steps 3 > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep_c5.err; echo "sweep rc=$?" >> gpurun_out/rc_c5.txt
