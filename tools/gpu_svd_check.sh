# GPU call: parity tests (both SVD back-ends) + bench with each back-end
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -x -q -rA -k "reduced_env or entrywise or iterations" > gpurun_out/pytest_svd.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc2.txt
timeout 600 python bench.py --svd gram --steps 10 --no-cpu-baseline > gpurun_out/bench_gram.json 2> gpurun_out/bench_gram.err; echo "bench gram rc=$?" >> gpurun_out/rc2.txt
