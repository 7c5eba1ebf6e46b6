#!/bin/bash
# A/B: in-cluster split-K vs slab + reduction kernel (both with the fused epilogues)
cd "$(dirname "$0")/.."
O=gpurun_out/n
mkdir -p $O
CTM_TC_SPLIT=slab timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "absorb or reduced_env or side_isometry or entrywise" > $O/pytest_slab.log 2>&1; echo "pytest slab rc=$?" >> $O/rc.txt
for r in 1 2; do
  for m in cluster slab; do
    CTM_TC_SPLIT=$m timeout 600 python bench.py --no-cpu-baseline > $O/bench_${m}_$r.json 2> $O/bench_${m}_$r.err; echo "bench $m $r rc=$?" >> $O/rc.txt
  done
done
