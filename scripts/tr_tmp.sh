python scripts/ab_env.py 16384 10 '' 2>/dev/null
AB_SEED=4 python scripts/ab_env.py 13000 10 '' 2>/dev/null
AB_SEED=4 python scripts/ab_env.py 5000 10 '' 2>/dev/null
