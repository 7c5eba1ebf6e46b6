# A/B an environment knob of the ISO solver on the C4/C5 sweep:  KNOB=CTM_ISO_RR1 VALUES="1 2 3"
mkdir -p gpurun_out; : > gpurun_out/knob.jsonl
for v in $VALUES; do
  env $KNOB=$v timeout 600 python tools/sweep.py --configs ${SWEEP:-c4,c5} --steps 5 | sed "s/^/{\"$KNOB\": \"$v\", \"r\": /; s/$/}/" >> gpurun_out/knob.jsonl
done
