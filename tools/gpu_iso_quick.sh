# Quick ISO-solver iteration loop: kernel microbench, ISO parity tests, C4 (+C5) move timing.
mkdir -p gpurun_out
rm -f gpurun_out/rc_q.txt
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -lineinfo -std=c++17 -I paper_2306_08212_b200/csrc \
  tools/bench_iso_kernels.cu -o gpurun_out/bench_iso_kernels && \
  for n in ${BIK_SIZES:-128 160}; do timeout 120 gpurun_out/bench_iso_kernels $n; done > gpurun_out/bik.txt 2>&1
echo "microbench rc=$?" >> gpurun_out/rc_q.txt
timeout 1500 python -m pytest tests -m gpu -q -x -k "${PYK:-iso}" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc_q.txt
timeout 900 python tools/sweep.py --configs ${SWEEP:-c4} --steps 5 > gpurun_out/sweep_q.jsonl 2> gpurun_out/sweep_q.err; echo "sweep rc=$?" >> gpurun_out/rc_q.txt
if [ -n "$A_B" ]; then CTM_ISO_TRSM=1 timeout 900 python tools/sweep.py --configs ${SWEEP:-c4} --steps 5 > gpurun_out/sweep_q_b.jsonl 2>> gpurun_out/sweep_q.err; fi
