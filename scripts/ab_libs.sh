for n in 16384 8192 4096; do
for lib in paper_1510_01041_b200/_lib ab_libs/rb5 ab_libs/rb6; do
  LMSB_LIB_PATH=$lib/liblmsb200.so timeout 120 python scripts/quick_time.py $n 12 2>&1 | tail -8 | python -c "
import json,sys
L=[json.loads(l) for l in sys.stdin if l.startswith('{')]
import statistics
print('$n', '$lib', round(statistics.median(d['ms_total'] for d in L),4), L[-1]['i'], L[-1]['j'])"
done; done
