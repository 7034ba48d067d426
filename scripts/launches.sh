#!/bin/bash
# Launch list (ncu, serialised) of one config-2 and one config-3 fit: per-kernel times.
# usage: bash scripts/launches.sh TAG
tag=${1:-dev}
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c2_${tag}.csv \
    python scripts/quick_time.py 16384 2 > gpurun_out/launch_c2_${tag}.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launch_c3_${tag}.csv \
    python scripts/quick_time.py 65536 1 > gpurun_out/launch_c3_${tag}.log 2>&1
python scripts/launch_summary.py gpurun_out/launch_c2_${tag}.csv > gpurun_out/launch_c2_${tag}.txt 2>&1
python scripts/launch_summary.py gpurun_out/launch_c3_${tag}.csv > gpurun_out/launch_c3_${tag}.txt 2>&1
head -40 gpurun_out/launch_c2_${tag}.txt; head -40 gpurun_out/launch_c3_${tag}.txt
