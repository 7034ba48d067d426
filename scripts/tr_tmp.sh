ncu --metrics gpu__time_duration.sum --clock-control none -k regex:line_wqa --csv python scripts/quick_time.py 16384 1 2>/dev/null | grep line_wqa | tail -1
python scripts/ab_env.py 16384 12 '' 'LMSB_SLOPE_BOUND=0' 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_lms.py -m gpu -x -q -k "slope or golden" 2>&1 | tail -2
