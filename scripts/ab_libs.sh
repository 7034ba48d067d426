#!/bin/bash
# Dev helper: config 2 / 3 timings for each library variant given (run under gpurun).
for lib in "$@"; do
  echo "== $lib"
  LMSB_LIB_PATH=$lib timeout 300 python scripts/quick_time.py ${N:-16384} ${REPS:-4} | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: round(d[k],3) if isinstance(d[k], float) else d[k] for k in ('ms_total','ms_collect','ms_partition','ms_bound','ms_band_filter','i','j')})"
done
