#!/bin/bash
# A/B: base vs current (cluster split-K) vs current (slab split-K), fused epilogues hoisted
cd "$(dirname "$0")/.."
O=gpurun_out/r
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "absorb or reduced_env or side_isometry or entrywise or iterations" > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
for r in 1 2; do
  CTM_LIB_PATH=$PWD/ab/libctm_r02base.so timeout 600 python bench.py --no-cpu-baseline > $O/bench_base_$r.json 2> $O/bench_base_$r.err; echo "bench base $r rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_cluster_$r.json 2> $O/bench_cluster_$r.err; echo "bench cluster $r rc=$?" >> $O/rc.txt
  CTM_TC_SPLIT=slab timeout 600 python bench.py --no-cpu-baseline > $O/bench_slab_$r.json 2> $O/bench_slab_$r.err; echo "bench slab $r rc=$?" >> $O/rc.txt
done
