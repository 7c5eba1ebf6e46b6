# GPU call: contraction parity + bench + launch list of the contraction-only move
mkdir -p gpurun_out
rm -f gpurun_out/rc5.txt
timeout 900 python -m pytest tests -m gpu -x -q -k "absorb or entrywise or injected or no_truncation or directional" > gpurun_out/pytest_gemm.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc5.txt
timeout 600 python bench.py --steps 10 --no-cpu-baseline > gpurun_out/bench_gemm.json 2> gpurun_out/bench_gemm.err; echo "bench rc=$?" >> gpurun_out/rc5.txt
timeout 300 python tools/prof_move.py c4 inject > gpurun_out/plain.log 2>&1 && timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size,l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum,sm__inst_executed_pipe_tensor_subpipe_dmma.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_gemm.csv python tools/prof_move.py c4 inject > gpurun_out/ncu_gemm.log 2>&1; echo "ncu rc=$?" >> gpurun_out/rc5.txt
