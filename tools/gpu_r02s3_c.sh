#!/bin/bash
# Round-2 session 3: fused filter GEMM (fgemm.cuh) -- parity subset, A/B against the tc_gemm + combine path
cd "$(dirname "$0")/.."
O=gpurun_out/s3c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "side_isometry_projectors or iterations_gauge_invariant or converge" > $O/pytest_quick.log 2>&1; echo "pytest quick rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --libs "base=@CTM_ISO_FGEMM=0,fg=" --procs 3 --moves 10 > $O/ab.jsonl 2> $O/ab.err; echo "ab rc=$?" >> $O/rc.txt
CTM_ISO_DEBUG=1 timeout 300 python tools/iso_debug_move.py c4 > $O/iso_fg.txt 2>&1
timeout 1500 python tools/ab_move.py --config c5 --libs "base=@CTM_ISO_FGEMM=0,fg=" --procs 2 --moves 4 > $O/ab_c5.jsonl 2> $O/ab_c5.err; echo "ab c5 rc=$?" >> $O/rc.txt
timeout 1500 python tools/ab_move.py --config c3 --libs "base=@CTM_ISO_FGEMM=0,fg=" --procs 2 --moves 10 > $O/ab_c3.jsonl 2> $O/ab_c3.err; echo "ab c3 rc=$?" >> $O/rc.txt
