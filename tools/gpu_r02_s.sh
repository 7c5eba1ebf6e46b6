#!/bin/bash
# A/B: base vs current vs current without the fused Chebyshev epilogue (CTM_ISO_NOFUSE)
cd "$(dirname "$0")/.."
O=gpurun_out/s
mkdir -p $O
for r in 1 2; do
  CTM_LIB_PATH=$PWD/ab/libctm_r02base.so timeout 600 python bench.py --no-cpu-baseline > $O/bench_base_$r.json 2> $O/bench_base_$r.err; echo "bench base $r rc=$?" >> $O/rc.txt
  timeout 600 python bench.py --no-cpu-baseline > $O/bench_cluster_$r.json 2> $O/bench_cluster_$r.err; echo "bench cluster $r rc=$?" >> $O/rc.txt
  CTM_ISO_NOFUSE=1 timeout 600 python bench.py --no-cpu-baseline > $O/bench_nofuse_$r.json 2> $O/bench_nofuse_$r.err; echo "bench nofuse $r rc=$?" >> $O/rc.txt
  CTM_ISO_NOFUSE=1 CTM_TC_SPLIT=slab timeout 600 python bench.py --no-cpu-baseline > $O/bench_nofuse_slab_$r.json 2> $O/bench_nofuse_slab_$r.err; echo "bench nofuse slab $r rc=$?" >> $O/rc.txt
done
