#!/bin/bash
# Dev helper (run under gpurun): fit times of alternative builds (LMSB_LIB_PATH).
# usage: ab_libs.sh "N ..." lib_dir ...
ns=$1; shift
for n in $ns; do for lib in paper_1510_01041_b200/_lib "$@"; do
  LMSB_LIB_PATH=$lib/liblmsb200.so timeout 120 python scripts/quick_time.py $n 12 2>&1 | python -c "
import json,sys,statistics
L=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print($n, '$lib', round(statistics.median(d['ms_total'] for d in L[2:]),4), L[-1]['i'], L[-1]['j'])"
done; done
