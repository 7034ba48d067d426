python scripts/ab_env.py 16384 10 '' 2>&1 | tail -1
LMSB_TRACE=1 python scripts/trace_fit.py 16384 3 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_lms.py -m gpu -x -q -k "device_plan or golden or band_path or hybrid" 2>&1 | tail -2
