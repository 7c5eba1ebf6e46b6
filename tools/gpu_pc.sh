mkdir -p gpurun_out
CTM_ISO_NOPC=1 CTM_ISO_DEBUG=1 timeout 300 python tools/iso_debug_move.py c4 2 > gpurun_out/pc0.out 2> gpurun_out/pc0.err
CTM_ISO_DEBUG=1 timeout 300 python tools/iso_debug_move.py c4 2 > gpurun_out/pc1.out 2> gpurun_out/pc1.err
timeout 900 python -m pytest tests -m gpu -q -x -k "iso" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?" > gpurun_out/rc_q.txt
timeout 900 python tools/sweep.py --configs c4,c5 --steps 5 > gpurun_out/sweep_q.jsonl 2> gpurun_out/sweep_q.err
