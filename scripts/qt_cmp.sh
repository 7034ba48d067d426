#!/bin/bash
# Dev helper: quick_time under several env settings (run under gpurun).
# usage: N=16384 REPS=3 bash scripts/qt_cmp.sh "LMSB_BAND_COARSE=0" "LMSB_BAND_COARSE=1"
for cfg in "$@"; do
  echo "== $cfg"
  env $cfg timeout 300 python scripts/quick_time.py ${N:-16384} ${REPS:-3} | tail -2 | python -c "
import json,sys
for l in sys.stdin:
    d=json.loads(l); print({k: round(d[k],4) if isinstance(d[k], float) else d[k] for k in ('ms_total','ms_collect','ms_partition','ms_bound','ms_band_filter','bands_searched','bands_refined','band_survivors','survivors','seed_height','i','j')})"
done
