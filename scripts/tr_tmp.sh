python scripts/ab_env.py 16384 10 '' 2>/dev/null
LMSB_TRACE=1 python scripts/trace_fit.py 16384 3 2>&1 | tail -2
