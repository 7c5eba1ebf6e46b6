mkdir -p gpurun_out
timeout 1200 python tools/sweep.py --configs c2,c3,c4,c5,c5_256 --steps 5 > gpurun_out/sweep_D_chi.jsonl 2> gpurun_out/sweep_D_chi.err
timeout 900 python tools/sweep.py --configs c2,c3,c4 --strategies sequential,reduced,standard --steps 3 > gpurun_out/sweep_strat.jsonl 2> gpurun_out/sweep_strat.err
echo done > gpurun_out/rc_sw.txt
