#!/bin/bash
# ISO solver knobs III around the re-tuned defaults (C4)
cd "$(dirname "$0")/.."
O=gpurun_out/s2o
mkdir -p $O
timeout 3000 python tools/ab_move.py --libs "base=,s1_12=@CTM_ISO_SAFE1=1.2,s_10=@CTM_ISO_SAFE=1.0,s_105=@CTM_ISO_SAFE=1.05,t3=@CTM_ISO_TAIL=3,t5=@CTM_ISO_TAIL=5,pw3=@CTM_ISO_POWER=3,pw5=@CTM_ISO_POWER=5,sw2=@CTM_ISO_SWEEPS1=2,gf64=@CTM_ISO_GFORM=64,spr5=@CTM_ISO_SPREAD=1e5,s12s105=@CTM_ISO_SAFE1=1.2@CTM_ISO_SAFE=1.05" --procs 3 --moves 12 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
