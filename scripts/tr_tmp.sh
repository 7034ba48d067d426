for lib in paper_1510_01041_b200/_lib/liblmsb200.so paper_1510_01041_b200/_lib/p2048/liblmsb200.so paper_1510_01041_b200/_lib/p4096/liblmsb200.so; do
LMSB_LIB_PATH=$lib python scripts/ab_env.py 16384 12 '' 2>&1 | tail -1 | cut -c1-120
LMSB_LIB_PATH=$lib python scripts/ab_env.py 65536 3 '' 2>&1 | tail -1 | cut -c1-250
done
