#!/bin/bash
# Round-2 session 3: fgemm also for the Ritz vectors (U = Y W, P W), the locked-space projection and the start
cd "$(dirname "$0")/.."
O=gpurun_out/s3d
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "side_isometry_projectors or iterations_gauge_invariant or converge" > $O/pytest_quick.log 2>&1; echo "pytest quick rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "prev=ab/libctm_fg1.so,new=" --procs 3 --moves 10 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c5 --libs "prev=ab/libctm_fg1.so,new=" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "prev=ab/libctm_fg1.so,new=" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
