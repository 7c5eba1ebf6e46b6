mkdir -p gpurun_out
bash tools/gpu_prof_full_move.sh
timeout 900 python tools/sweep.py --configs c2,c3,c4 --strategies sequential,reduced,standard --steps 3 > gpurun_out/sweep_strat.jsonl 2> gpurun_out/sweep_strat.err
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu0.log 2>&1; echo "ncu bench rc=$?" > gpurun_out/rc_r2.txt
