#!/bin/bash
# Round profile (run under gpurun): ncu summaries of the config-2 band kernels,
# the config-3 large-n kernels, the fused small-fit kernel and the device
# detect kernels; launch lists of configs 2, 3 and 5; then the default bench
# lines (ours and the reference arm).  usage: bash scripts/profile_round.sh TAG
set -x
tag=${1:-r02}
mkdir -p gpurun_out
ncu --set full --clock-control none --import-source on \
    -k regex:"band_filter_kernel|band_bound_kernel|sweep_enum|sweep_classify|band_count_kernel|exact_cached|exact_cluster|sub_scatter|band_prepass_count" \
    -o gpurun_out/${tag}_band python scripts/quick_time.py 16384 1 > gpurun_out/ncu_band.log 2>&1
python scripts/ncu_summary.py gpurun_out/${tag}_band.ncu-rep profiles/${tag}_band_kernels_ncu.json
ncu --set full --clock-control none -k regex:"band_filter_big|sweep_enum|sweep_classify|band_prepass_count|band_coarse|exact_cluster|seg_sort" -c 8 \
    -o gpurun_out/${tag}_big python scripts/quick_time.py 65536 1 > gpurun_out/ncu_big.log 2>&1
python scripts/ncu_summary.py gpurun_out/${tag}_big.ncu-rep profiles/${tag}_big_kernels_ncu.json
ncu --set full --clock-control none -k regex:small_fit -c 1 \
    -o gpurun_out/${tag}_small python scripts/quick_batch.py 2048 512 1 > gpurun_out/ncu_small.log 2>&1
python scripts/ncu_summary.py gpurun_out/${tag}_small.ncu-rep profiles/${tag}_small_fit_ncu.json small_fit
ncu --set full --clock-control none -k regex:"img_vote|support_count_img|support_write_img|peaks_kernel" \
    -o gpurun_out/${tag}_detect python scripts/detect_once.py 1 > gpurun_out/ncu_detect.log 2>&1
python scripts/ncu_summary.py gpurun_out/${tag}_detect.ncu-rep profiles/${tag}_detect_ncu.json
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_config2.csv \
    python bench.py --steps 2 --warmup 1 --no-extra --no-cpu-baseline > gpurun_out/bench_under_ncu.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_launches_config3.csv \
    python scripts/quick_time.py 65536 1 > gpurun_out/ncu_c3.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/${tag}_launches_config5.csv python scripts/detect_once.py 1 > gpurun_out/ncu_c5.log 2>&1
cp profiles/${tag}_*_ncu.json gpurun_out/
python bench.py > gpurun_out/bench_${tag}.json 2> gpurun_out/bench_${tag}.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_${tag}.json 2> gpurun_out/bench_ref_${tag}.err
tail -c 4000 gpurun_out/bench_${tag}.json
cat gpurun_out/bench_ref_${tag}.json
# the full reports stay on the box (gpurun copies back at most 64 MiB)
rm -f gpurun_out/*.ncu-rep
