#!/bin/bash
# Round-2 session 3, last: full GPU suite, smoke, bench and reference arm after the pinned round-trip change
cd "$(dirname "$0")/.."
O=gpurun_out/f7
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 2400 python -m pytest tests -m gpu -q -rA -s --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python tools/sweep.py --configs c2,c3,c4,c5,c5_256 --strategies sequential --steps 5 > $O/sweep_seq.jsonl 2> $O/sweep.err; echo "sweep rc=$?" >> $O/rc.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu0.log 2>&1; echo "ncu bench launches rc=$?" >> $O/rc.txt
