#!/bin/bash
# Dev helper: config 4 batch timings for each library variant given (run under gpurun).
for lib in "$@"; do
  echo "== $lib"
  LMSB_LIB_PATH=$lib timeout 300 python scripts/quick_batch.py ${F:-8192} ${NB:-512} 3 | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: d[k] for k in ('ms_total','survivors','band_survivors','r0')})"
done
