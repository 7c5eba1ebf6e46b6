#!/bin/bash
# Round-2 session 3: one pinned round trip per convergence check (status + Ritz values + residuals)
cd "$(dirname "$0")/.."
O=gpurun_out/s3o
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py -q -x -k "golden or side_isometry_projectors or main_ts or side_ts or iterations_gauge or non_finite or errors" > $O/pytest_quick.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
L="prev=ab/libctm_prev.so,new="
timeout 1500 python tools/ab_move.py --libs "$L" --procs 4 --moves 10 > $O/ab_c4.jsonl 2> $O/ab_c4.err; echo "ab c4 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "$L" --procs 3 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "$L" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c2 --libs "$L" --procs 3 --moves 10 > $O/ab_c2.jsonl 2> $O/ab_c2.err; echo "ab c2 rc=$?" >> $O/rc.txt
