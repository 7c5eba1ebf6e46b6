#!/bin/bash
# Round-2 session 3: fgemm with a second k-group of warps per CTA (FG_KSPLIT=2), 3 and 4 stages
cd "$(dirname "$0")/.."
O=gpurun_out/s3k
mkdir -p $O
L="base=,ks2=ab/libctm_ks2.so,ks2st4=ab/libctm_ks2_st4.so"
timeout 1500 python tools/ab_move.py --libs "$L" --procs 3 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
CTM_LIB_PATH=ab/libctm_ks2.so timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "golden or side_isometry_projectors or main_ts or side_ts" > $O/pytest_ks2.log 2>&1; echo "pytest ks2 rc=$?" >> $O/rc.txt
