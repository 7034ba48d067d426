LMSB_TRACE=1 python scripts/trace_fit.py 16384 3 2>&1 | tail -2
python scripts/ab_env.py 16384 8 'LMSB_GROUP_MODE=1' 'LMSB_GROUP_MODE=3' 'LMSB_SUB_SAMPLES=2' 'LMSB_BAND_CHUNK=8192' 'LMSB_BAND_CHUNK=16384'
AB_SEED=3 python scripts/ab_env.py 20000 6 'LMSB_GROUP_MODE=1' 'LMSB_GROUP_MODE=3'
AB_SEED=4 python scripts/ab_env.py 13000 6 'LMSB_GROUP_MODE=1' 'LMSB_GROUP_MODE=3'
timeout 900 python -m pytest tests/test_gpu_lms.py -m gpu -x -q 2>&1 | tail -3
