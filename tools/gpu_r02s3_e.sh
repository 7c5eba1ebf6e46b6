#!/bin/bash
# Round-2 session 3: CTM_FLAG_WARM_START first measurements
cd "$(dirname "$0")/.."
O=gpurun_out/s3e
mkdir -p $O
timeout 600 python tools/warm_moves.py c4 12 > $O/warm_c4.jsonl 2> $O/warm_c4.err; echo "warm c4 rc=$?" >> $O/rc.txt
CTM_ISO_DEBUG=1 timeout 600 python tools/warm_moves.py c4 4 > /dev/null 2> $O/warm_c4_debug.txt; echo "warm c4 debug rc=$?" >> $O/rc.txt
timeout 600 python tools/warm_moves.py c3 6 iterate > $O/warm_c3_iter.jsonl 2> $O/warm_c3.err; echo "warm c3 rc=$?" >> $O/rc.txt
timeout 600 python tools/warm_moves.py c5 6 > $O/warm_c5.jsonl 2> $O/warm_c5.err; echo "warm c5 rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -s -k "c2-20-True or golden or warm_start" > $O/pytest_warm.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
