#!/bin/bash
# Round check (run under gpurun): the whole GPU suite, then the round profile
# (ncu summaries, launch lists, bench lines).  usage: bash scripts/round_check.sh TAG
tag=${1:-r02}
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1
tail -3 gpurun_out/pytest_gpu.log
bash scripts/profile_round.sh $tag > gpurun_out/profile_round.log 2>&1
tail -c 1500 gpurun_out/bench_${tag}.json
