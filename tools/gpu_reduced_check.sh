mkdir -p gpurun_out
rm -f gpurun_out/rc6.txt
timeout 900 python -m pytest tests -m gpu -q -rA -k "reduced_env_exact or reduced_move" > gpurun_out/pytest_red.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc6.txt
timeout 1500 python tools/sweep.py --configs c2,c3,c4 --steps 3 --strategies reduced,sequential > gpurun_out/sweep_red.jsonl 2> gpurun_out/sweep_red.err; echo "sweep rc=$?" >> gpurun_out/rc6.txt
