python scripts/ab_env.py 16384 12 'LMSB_GRAPH=0' 'LMSB_GRAPH=1' 2>&1 | tail -2
AB_SEED=4 python scripts/ab_env.py 5000 12 'LMSB_GRAPH=0' 'LMSB_GRAPH=1' 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_lms.py -m gpu -x -q -k "device_plan or golden or hybrid or deferred or slope" 2>&1 | tail -2
