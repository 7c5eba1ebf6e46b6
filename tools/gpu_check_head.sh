#!/bin/bash
# sanity check of HEAD on a B200: GPU suite + bench
cd "$(dirname "$0")/.."
O=gpurun_out/${1:-head}
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 600 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 1500 python -m pytest tests -m gpu -x -q -rA --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
