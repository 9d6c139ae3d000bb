#!/bin/bash
# C5 partitioning at scale: RMAT-30 in 8 partitions on one B200, BFS certificate.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g > gpurun_out/r3h.log
TG_RMAT30=1 timeout 1500 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k "rmat30_pagerank_one_gpu and 8" --durations=3 >> gpurun_out/r3h.log 2>&1
tail -8 gpurun_out/r3h.log
