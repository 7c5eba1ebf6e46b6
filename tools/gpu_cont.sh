mkdir -p gpurun_out; : > gpurun_out/cont.jsonl
for cm in 1 2 99; do
  CTM_ISO_CONT_MIN=$cm timeout 600 python tools/sweep.py --configs c4,c5 --steps 5 | sed "s/^/{\"cont_min\": $cm, \"r\": /; s/$/}/" >> gpurun_out/cont.jsonl
done
for cm in 2 99; do CTM_ISO_CONT_MIN=$cm CTM_ISO_DEBUG=1 timeout 300 python tools/iso_debug_move.py c5 2 > /dev/null 2> gpurun_out/isodbg5_$cm.err; done
