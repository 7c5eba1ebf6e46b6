#!/bin/bash
# Round-2 session 3: re-check the restored tree (smoke, bench) and A/B the oversampling at C4
cd "$(dirname "$0")/.."
O=gpurun_out/s3a
mkdir -p $O
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py --no-cpu-baseline > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "base=,p48=@CTM_ISO_P=48" --procs 3 --moves 10 > $O/ab_p.jsonl 2> $O/ab_p.err; echo "ab rc=$?" >> $O/rc.txt
CTM_ISO_DEBUG=1 CTM_ISO_P=48 timeout 300 python tools/iso_debug_move.py c4 > $O/iso_p48.txt 2>&1
CTM_ISO_DEBUG=1 timeout 300 python tools/iso_debug_move.py c4 > $O/iso_p32.txt 2>&1
