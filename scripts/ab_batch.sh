#!/bin/bash
# Dev helper (run under gpurun): config-4 batch device time of alternative builds.
# usage: ab_batch.sh lib_dir ...
for lib in paper_1510_01041_b200/_lib "$@"; do
  LMSB_LIB_PATH=$lib/liblmsb200.so timeout 300 python scripts/quick_batch.py 8192 512 5 2>&1 | python -c "
import json,sys,statistics
L=[json.loads(l) for l in sys.stdin if l.startswith('{')]
print('$lib', round(statistics.median(d['ms_total'] for d in L[1:]),3), L[-1]['r0'], L[-1]['found'])"
done
