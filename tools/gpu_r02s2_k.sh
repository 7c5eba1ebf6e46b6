#!/bin/bash
# ISO solver tuning knobs re-measured after the Jacobi / Cholesky changes (C4 full move A/B)
cd "$(dirname "$0")/.."
O=gpurun_out/s2k
mkdir -p $O
timeout 3000 python tools/ab_move.py --libs "base=,p24=@CTM_ISO_P=24,p16=@CTM_ISO_P=16,s1_16=@CTM_ISO_SAFE1=1.6,s1_25=@CTM_ISO_SAFE1=2.5,s_11=@CTM_ISO_SAFE=1.1,s_15=@CTM_ISO_SAFE=1.5,tail4=@CTM_ISO_TAIL=4,tail8=@CTM_ISO_TAIL=8,sp8=@CTM_ISO_SPREAD_PLAIN=1e8,sp12=@CTM_ISO_SPREAD_PLAIN=1e12" --procs 3 --moves 12 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
