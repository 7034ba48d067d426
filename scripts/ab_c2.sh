#!/bin/bash
# Dev helper (run under gpurun): config 2 / 8,192 / config 3 fit times under knob variants
# (one process per variant; knobs read at launch time).  usage: ab_c2.sh 'K=V' ...
for n in 16384 8192 65536; do
for v in "$@"; do
  env $v timeout 120 python scripts/quick_time.py $n 12 2>&1 | python -c "
import json,sys,statistics
L=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print($n, '$v', round(statistics.median(d['ms_total'] for d in L[2:]),4), L[-1]['i'], L[-1]['j'], L[-1]['h'])"
done; done
