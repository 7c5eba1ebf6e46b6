mkdir -p gpurun_out
rm -f gpurun_out/rc6.txt
timeout 900 python -m pytest tests -m gpu -q -rA -k "reduced_env_exact or reduced_move" > gpurun_out/pytest_red.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc6.txt
CTM_ISO_DEBUG=1 timeout 1500 python tools/sweep.py --configs c2,c3,c4 --steps 2 --strategies standard > gpurun_out/sweep_std.jsonl 2> gpurun_out/sweep_std.err; echo "sweep rc=$?" >> gpurun_out/rc6.txt
