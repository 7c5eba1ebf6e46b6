#!/bin/bash
# Round-2 session 3: solver knobs re-checked after the faster fgemm (filter degrees got cheaper relative to checks)
cd "$(dirname "$0")/.."
O=gpurun_out/s3l
mkdir -p $O
L="base=,safe1_16=@CTM_ISO_SAFE1=1.6,safe_12=@CTM_ISO_SAFE=1.2,tail3=@CTM_ISO_TAIL=3,power3=@CTM_ISO_POWER=3,power2=@CTM_ISO_POWER=2"
timeout 1500 python tools/ab_move.py --libs "$L" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
