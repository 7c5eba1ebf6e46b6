# End-of-round GPU evidence: smoke, full GPU suite, default bench, launch list, ncu full capture
mkdir -p gpurun_out
rm -f gpurun_out/rcf.txt
nvidia-smi > gpurun_out/final_nvsmi.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/rcf.txt
timeout 1800 python -m pytest tests -m gpu -q -rA > gpurun_out/final_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rcf.txt
timeout 900 python bench.py > gpurun_out/final_bench.json 2> gpurun_out/final_bench.err; echo "bench rc=$?" >> gpurun_out/rcf.txt
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/final_bench_ref.json 2> gpurun_out/final_bench_ref.err; echo "bench ref rc=$?" >> gpurun_out/rcf.txt
CTM_BENCH_PROFILE=1 timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final_launches_bench.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/final_ncu0.log 2>&1; echo "ncu bench launches rc=$?" >> gpurun_out/rcf.txt
timeout 300 python tools/prof_move.py c4 inject > gpurun_out/plain.log 2>&1 && timeout 900 ncu --profile-from-start off --metrics gpu__time_duration.sum,launch__grid_size --clock-control none --csv --log-file gpurun_out/final_launches.csv python tools/prof_move.py c4 inject > gpurun_out/final_ncu1.log 2>&1; echo "ncu launches rc=$?" >> gpurun_out/rcf.txt
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none -k regex:tc_gemm -c 6 -o gpurun_out/final_prof_tcgemm python tools/prof_move.py c4 inject > gpurun_out/final_ncu2.log 2>&1; echo "ncu full rc=$?" >> gpurun_out/rcf.txt
