mkdir -p gpurun_out
SWEEP=c4,c5 BIK_SIZES="96 128 160" bash tools/gpu_iso_quick.sh
