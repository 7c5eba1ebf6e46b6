#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
out=gpurun_out/r02_knobs_rr.jsonl
: > $out
for p in 2 1 2 1; do
  CTM_ISO_RR_PASSES=$p timeout 300 python bench.py --no-cpu-baseline --steps 10 > /tmp/k.json 2>/dev/null
  python - "$p" >> $out <<'PY'
import json, sys
d = json.loads(open('/tmp/k.json').read().strip().splitlines()[-1])
print(json.dumps({"rr_passes": sys.argv[1], "ms": d["ms_per_step"], "iso": d["solver"]["ms_isometry_stage_per_move"], "fallbacks": d["svd_fallbacks_per_move"]}))
PY
done
CTM_ISO_RR_PASSES=1 timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -x -k "main_ts or side_ts or shadowed_trajectory and c3" > gpurun_out/r02_rr1_pytest.log 2>&1
echo "pytest exit $?" >> gpurun_out/r02_rr1_pytest.log
CTM_ISO_RR_PASSES=1 CTM_ISO_DEBUG=1 timeout 600 python tools/iso_fallback_debug.py c3 8 > gpurun_out/r02_rr1_c3_moves.txt 2>/dev/null
