mkdir -p gpurun_out
rm -f gpurun_out/rc3.txt
timeout 900 python -m pytest tests -m gpu -q -rA -k "iso" > gpurun_out/pytest_iso.log 2>&1; echo "pytest rc=$?" >> gpurun_out/rc3.txt
CTM_ISO_DEBUG=1 timeout 600 python bench.py --svd iso --steps 10 --no-cpu-baseline > gpurun_out/bench_iso.json 2> gpurun_out/bench_iso.err; echo "bench iso rc=$?" >> gpurun_out/rc3.txt
