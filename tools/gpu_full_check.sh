mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" > gpurun_out/rc_full.txt
timeout 900 python tools/sweep.py --configs ${SWEEP:-c4,c5,c5_256} --steps 5 > gpurun_out/sweep_q.jsonl 2> gpurun_out/sweep_q.err; echo "sweep rc=$?" >> gpurun_out/rc_full.txt
CTM_ISO_DEBUG=1 timeout 300 python tools/iso_debug_move.py c4 2 > /dev/null 2> gpurun_out/isodbg4.err
