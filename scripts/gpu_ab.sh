#!/bin/bash
# Dev helper (run under gpurun): knob A/B on configs 2 and 3, then the band tests.
set -x
timeout 300 python scripts/ab_env.py 16384 12 'LMSB_BAND_GROUP=0' 'LMSB_BAND_GROUP=1' 'LMSB_SUB_SAMPLES=2' 'LMSB_SUB_SAMPLES=4' > gpurun_out/ab_c2.log 2>&1
AB_SEED=1 timeout 300 python scripts/ab_env.py 8192 12 'LMSB_BAND_GROUP=0' 'LMSB_BAND_GROUP=1' 'LMSB_SUB_SAMPLES=2' > gpurun_out/ab_8k.log 2>&1
cat gpurun_out/ab_c2.log gpurun_out/ab_8k.log
timeout 900 python -m pytest tests/test_gpu_lms.py -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_lms.log 2>&1
tail -5 gpurun_out/pytest_lms.log
