mkdir -p gpurun_out
nvidia-smi > gpurun_out/nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rc.txt
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc.txt
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench rc=$?" >> gpurun_out/rc.txt
timeout 300 python tools/prof_move.py c4 inject > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/launches.csv python tools/prof_move.py c4 inject > gpurun_out/ncu1.log 2>&1; echo "ncu1 rc=$?" >> gpurun_out/rc.txt
timeout 900 ncu --set full --clock-control none --import-source on -k regex:tc_gemm -s 70 -c 8 -o gpurun_out/prof_tcgemm python tools/prof_move.py c4 inject > gpurun_out/ncu2.log 2>&1; echo "ncu2 rc=$?" >> gpurun_out/rc.txt
