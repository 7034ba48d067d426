#!/bin/bash
# Dev helper (run under gpurun): simulated scaling of configs 3 and 2 under knob variants.
for v in "$@"; do
  echo "== $v"
  env $v timeout 300 python scripts/sim_scaling.py 65536 3 | python -c "
import json,sys
for l in sys.stdin:
  d=json.loads(l); print(d['R'], d['one_gpu_ms'], d['owned_max_ms'], d['same_record'], max(r['plan_ms'] for r in d['ranks']), max(r['search_ms'] for r in d['ranks']))"
done
