#!/bin/bash
# Round-2 (session 3, after the fgemm solver GEMMs) end-of-round GPU evidence for the current code
cd "$(dirname "$0")/.."
O=gpurun_out/f6
mkdir -p $O
nvidia-smi > $O/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?" >> $O/rc.txt
timeout 900 python bench.py > $O/bench.json 2> $O/bench.err; echo "bench rc=$?" >> $O/rc.txt
timeout 900 python bench.py --impl reference --steps 2 --warmup 0 > $O/bench_ref.json 2> $O/bench_ref.err; echo "bench ref rc=$?" >> $O/rc.txt
timeout 300 python tools/prof_move.py c4 inject > /dev/null 2>&1
timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/launches_inject.csv python tools/prof_move.py c4 inject > $O/ncu1.log 2>&1; echo "ncu inject rc=$?" >> $O/rc.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file $O/launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu0.log 2>&1; echo "ncu bench launches rc=$?" >> $O/rc.txt
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:tc_gemm -s 2 -c 1 -o $O/prof_tcgemm_s3 python tools/prof_move.py c4 inject > $O/ncu2.log 2>&1; echo "ncu full tc_gemm rc=$?" >> $O/rc.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:chol_kernel -s 20 -c 1 -o $O/prof_chol python bench.py --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu3.log 2>&1; echo "ncu full chol rc=$?" >> $O/rc.txt
timeout 2700 python -m pytest tests -m gpu -q -rA -s --durations=20 > $O/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $O/rc.txt
timeout 1500 python tools/sweep.py --configs c2,c3,c4,c5,c5_256 --strategies sequential --steps 5 > $O/sweep_seq.jsonl 2> $O/sweep.err; echo "sweep rc=$?" >> $O/rc.txt
timeout 600 python tools/trace_move.py c4 > $O/trace_summary.txt 2>&1; echo "trace rc=$?" >> $O/rc.txt
