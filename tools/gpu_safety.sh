mkdir -p gpurun_out; : > gpurun_out/safety.jsonl
for sf in 1.25 1.0 0.85 0.7; do
  CTM_ISO_SAFETY=$sf timeout 600 python tools/sweep.py --configs c4,c5 --steps 5 | sed "s/^/{\"safety\": $sf, \"r\": /; s/$/}/" >> gpurun_out/safety.jsonl
done
