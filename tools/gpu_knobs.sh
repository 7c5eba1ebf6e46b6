#!/bin/bash
# A/B knobs on the C4 bench: CTM_GEMM_SHARE, CTM_ISO_FLAT_SAFETY
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/r02_knobs.jsonl
: > $out
for cfg in "1 2.0" "2 2.0" "4 2.0" "8 2.0"; do
  set -- $cfg
  CTM_GEMM_SHARE=$1 CTM_ISO_FLAT_SAFETY=$2 timeout 300 python bench.py --no-cpu-baseline --steps 10 > /tmp/k.json 2>/dev/null
  python - "$1" "$2" >> $out <<'PY'
import json, sys
d = json.loads(open('/tmp/k.json').read().strip().splitlines()[-1])
print(json.dumps({"share": sys.argv[1], "flat_safety": sys.argv[2], "ms": d["ms_per_step"], "iso": d["solver"]["ms_isometry_stage_per_move"], "fallbacks": d["svd_fallbacks_per_move"]}))
PY
done
