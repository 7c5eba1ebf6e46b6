#!/bin/bash
# ISO solver knobs II: combinations around the first-plan safety factor, C4 and C5
cd "$(dirname "$0")/.."
O=gpurun_out/s2l
mkdir -p $O
timeout 2400 python tools/ab_move.py --libs "base=,s16=@CTM_ISO_SAFE1=1.6,s14=@CTM_ISO_SAFE1=1.4,s12=@CTM_ISO_SAFE1=1.2,s16s11=@CTM_ISO_SAFE1=1.6@CTM_ISO_SAFE=1.1,s16t4=@CTM_ISO_SAFE1=1.6@CTM_ISO_TAIL=4,s16s11t4=@CTM_ISO_SAFE1=1.6@CTM_ISO_SAFE=1.1@CTM_ISO_TAIL=4,s14s11t4=@CTM_ISO_SAFE1=1.4@CTM_ISO_SAFE=1.1@CTM_ISO_TAIL=4" --procs 3 --moves 12 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "base=,s16=@CTM_ISO_SAFE1=1.6,s16s11t4=@CTM_ISO_SAFE1=1.6@CTM_ISO_SAFE=1.1@CTM_ISO_TAIL=4" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 900 python tools/ab_move.py --config c3 --libs "base=,s16=@CTM_ISO_SAFE1=1.6,s16s11t4=@CTM_ISO_SAFE1=1.6@CTM_ISO_SAFE=1.1@CTM_ISO_TAIL=4" --procs 2 --moves 12 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
