#!/bin/bash
# A/B: per-launch priority and exclusive SMs for the solver's latency kernels (C4 bench)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/r02_knobs_latency.jsonl
: > $out
for cfg in "0 0" "1 0" "0 1" "1 1" "0 0"; do
  set -- $cfg
  CTM_PRIO=$1 CTM_EXCL=$2 timeout 300 python bench.py --no-cpu-baseline --steps 10 > /tmp/k.json 2>/dev/null
  python - "$1" "$2" >> $out <<'PY'
import json, sys
d = json.loads(open('/tmp/k.json').read().strip().splitlines()[-1])
print(json.dumps({"prio": sys.argv[1], "excl": sys.argv[2], "ms": d["ms_per_step"], "iso": d["solver"]["ms_isometry_stage_per_move"], "fallbacks": d["svd_fallbacks_per_move"]}))
PY
done
