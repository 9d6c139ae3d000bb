#!/bin/bash
# C5's graph on one B200: RMAT-30 BFS exact certificate + RMAT-30 PageRank sample recurrence (opt-in tests)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g > gpurun_out/r2ab_rmat30.log; nproc >> gpurun_out/r2ab_rmat30.log
TG_RMAT30=1 timeout 2700 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k rmat30 --durations=3 >> gpurun_out/r2ab_rmat30.log 2>&1
echo "rc=$?" >> gpurun_out/r2ab_rmat30.log
tail -15 gpurun_out/r2ab_rmat30.log
