#!/bin/bash
# Dev helper: band-size sweep on config 2 (run under gpurun).
for bv in ${BVS:-8192 16384 32768 65536 131072}; do
  echo "== LMSB_BAND_VERTICES=$bv"
  LMSB_BAND_VERTICES=$bv timeout 120 python scripts/quick_time.py 16384 3 | tail -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print({k: d[k] for k in ('ms_total','ms_bound','ms_partition','ms_band_filter','ms_exact','bands','bands_searched','filtered_vertices','survivors','seed_height','band_survivors','h')})"
done
