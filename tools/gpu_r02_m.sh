#!/bin/bash
# cluster split-K + fused Chebyshev epilogue + K7 warp-sum: parity subset, bench, cuBLAS comparison
cd "$(dirname "$0")/.."
O=gpurun_out/m
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench2.json 2> $O/bench2.err; echo "bench2 rc=$?" >> $O/rc.txt
timeout 300 python tools/cublas_steps.py > $O/cublas_steps.jsonl 2> $O/cublas.err; echo "cublas rc=$?" >> $O/rc.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu0.log 2>&1; echo "ncu rc=$?" >> $O/rc.txt
