#!/bin/bash
cd "$(dirname "$0")/.."
O=gpurun_out/v
mkdir -p $O
timeout 120 python tools/cublas_one.py 16384 1024 128 > /dev/null 2>&1
timeout 600 ncu --profile-from-start off --set full --clock-control none -o $O/cublas_s4 -f python tools/cublas_one.py 16384 1024 128 > $O/ncu_s4.log 2>&1; echo "s4 rc=$?" >> $O/rc.txt
timeout 600 ncu --profile-from-start off --set full --clock-control none -o $O/cublas_s3 -f python tools/cublas_one.py 16384 128 1024 > $O/ncu_s3.log 2>&1; echo "s3 rc=$?" >> $O/rc.txt
timeout 600 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:tc_gemm -s 3 -c 1 -o $O/tc_s4 -f python tools/prof_move.py c4 inject > $O/ncu_tc.log 2>&1; echo "tc rc=$?" >> $O/rc.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q > $O/pytest.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
