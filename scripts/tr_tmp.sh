python scripts/ab_env.py 16384 8 '' 'LMSB_GROUP_MODE=1'
python scripts/ab_env.py 65536 3 '' 'LMSB_BIG_NARROW=1'
