#!/bin/bash
# ncu --set full of the sweep enumeration kernel (config 2 and 3)
mkdir -p gpurun_out
tag=${1:-dev}
ncu --set full --clock-control none --import-source on -k regex:sweep_enum -c 1 -o gpurun_out/sweep_enum_c2_${tag} \
    python scripts/quick_time.py 16384 1 > gpurun_out/ncu_sweep_c2_${tag}.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:sweep_enum -c 1 -o gpurun_out/sweep_enum_c3_${tag} \
    python scripts/quick_time.py 65536 1 > gpurun_out/ncu_sweep_c3_${tag}.log 2>&1
