#!/bin/bash
# Round profile: ncu capture of the collect kernel, launch list of a short
# bench, then the default bench line (run under gpurun).
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:band_collect_kernel -c 1 \
    -o gpurun_out/r01_collect python scripts/quick_time.py 16384 1 > gpurun_out/ncu_collect.log 2>&1
python scripts/ncu_summary.py gpurun_out/r01_collect.ncu-rep profiles/r01_collect_ncu.json band_collect
cp profiles/r01_collect_ncu.json gpurun_out/
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_band.csv \
    python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 3000 gpurun_out/bench.json
