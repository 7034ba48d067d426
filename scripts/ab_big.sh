#!/bin/bash
# Dev helper (run under gpurun): large-n fit times under knob variants.  usage: ab_big.sh "N ..." 'K=V' ...
ns=$1; shift
for n in $ns; do for v in "$@"; do
  env $v timeout 120 python scripts/quick_time.py $n 7 2>&1 | python -c "
import json,sys,statistics
L=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print($n, '$v', round(statistics.median(d['ms_total'] for d in L[2:]),4), L[-1]['i'], L[-1]['j'], L[-1]['band_survivors'])"
done; done
