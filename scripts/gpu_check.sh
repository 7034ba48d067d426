#!/bin/bash
# Dev helper: GPU tests + quick timings (run under gpurun).
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 300 python scripts/quick_time.py 16384 3 > gpurun_out/qt_band.log 2>&1
LMSB_BAND=0 timeout 300 python scripts/quick_time.py 16384 2 > gpurun_out/qt_filter.log 2>&1
timeout 120 python scripts/quick_time.py 1000 3 > gpurun_out/qt_1000.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q ${PYTEST_ARGS} > gpurun_out/pytest_gpu.log 2>&1
tail -5 gpurun_out/pytest_gpu.log
cat gpurun_out/qt_*.log
