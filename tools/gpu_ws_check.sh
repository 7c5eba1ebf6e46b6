mkdir -p gpurun_out
rm -f gpurun_out/rc8.txt
CTM_DEBUG_WS=1 timeout 300 python tools/ws_sizes.py > gpurun_out/ws.txt 2>&1; echo "ws rc=$?" >> gpurun_out/rc8.txt
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/pytest_all2.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc8.txt
timeout 1500 python tools/sweep.py --steps 3 > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err; echo "sweep rc=$?" >> gpurun_out/rc8.txt
