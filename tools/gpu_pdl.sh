mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_full.log 2>&1; echo "pytest rc=$?" > gpurun_out/rc_full.txt
KNOB=CTM_NO_PDL VALUES="1" SWEEP=c3,c4,c5 bash tools/gpu_knob.sh; cp gpurun_out/knob.jsonl gpurun_out/knob_nopdl.jsonl
timeout 900 python tools/sweep.py --configs c3,c4,c5 --steps 5 > gpurun_out/knob_pdl.jsonl
