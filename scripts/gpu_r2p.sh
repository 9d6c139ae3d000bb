#!/bin/bash
# PageRank die split: parity, then A/B at RMAT-28
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "die" > gpurun_out/r2p_tests.log 2>&1; tail -3 gpurun_out/r2p_tests.log
O=gpurun_out/r2p_pr_sweep.txt
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_SPLIT=0;1" "TG_PR_HOT=16777216;33554432;67108864" > $O 2>&1
cat $O
