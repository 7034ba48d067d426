#!/bin/bash
# Dev helper (run under gpurun): per-stage trace of one rank's plan + owned search.
for R in 8 1; do for n in 65536 16384; do
  echo "== n $n rank 0 of $R"
  LMSB_TRACE=1 timeout 120 python scripts/owned_rank.py $n $R 0 2>&1 | grep trace_us | tail -3 | python -c "
import json,sys
for l in sys.stdin:
  t=json.loads(l)['trace_us']; print([(a,round(b)) for a,b in t][-24:])"
done; done
