timeout 1700 python -m pytest tests/test_gpu_lms.py -m gpu -x -q 2>&1 | tail -2
python scripts/ab_env.py 16384 12 '' 2>&1 | tail -1 | cut -c1-150
