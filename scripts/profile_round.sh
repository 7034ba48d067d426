#!/bin/bash
# Round profile: ncu captures of the band-stage kernels and the fused small-fit
# kernel, launch list of a short bench, then the default bench lines (run
# under gpurun).
set -x
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on -k regex:band_collect_kernel -c 1 \
    -o gpurun_out/r01_collect python scripts/quick_time.py 16384 1 > gpurun_out/ncu_collect.log 2>&1
python scripts/ncu_summary.py gpurun_out/r01_collect.ncu-rep profiles/r01_collect_ncu.json band_collect
ncu --set full --clock-control none -k regex:"band_filter_kernel|band_bound_kernel|band_count_kernel|exact_cached" \
    -o gpurun_out/r01_band_kernels python scripts/quick_time.py 16384 1 > gpurun_out/ncu_band.log 2>&1
python scripts/ncu_summary.py gpurun_out/r01_band_kernels.ncu-rep profiles/r01_band_kernels_ncu.json
ncu --set full --clock-control none -k regex:small_fit -c 1 \
    -o gpurun_out/r01_small python scripts/quick_batch.py 2048 512 1 > gpurun_out/ncu_small.log 2>&1
python scripts/ncu_summary.py gpurun_out/r01_small.ncu-rep profiles/r01_small_fit_ncu.json small_fit
ncu --set full --clock-control none -k regex:"band_coarse_kernel|band_filter_big_kernel|band_count_kernel" -c 3 \
    -o gpurun_out/r01_big python scripts/quick_time.py 65536 1 > gpurun_out/ncu_big.log 2>&1
python scripts/ncu_summary.py gpurun_out/r01_big.ncu-rep profiles/r01_big_kernels_ncu.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_config3.csv \
    python scripts/quick_time.py 65536 1 > gpurun_out/ncu_c3.log 2>&1
cp profiles/r01_*_ncu.json gpurun_out/
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r01_launches_band.csv \
    python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
tail -c 3000 gpurun_out/bench.json
