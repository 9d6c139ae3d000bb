#!/bin/bash
# PageRank hub split: parity, then K sweep at RMAT-28
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "hub_split or variants or ghost_pull" > gpurun_out/r2m_tests.log 2>&1; tail -3 gpurun_out/r2m_tests.log
O=gpurun_out/r2m_pr_sweep.txt
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_HUB=0;16384;32768;49152;53248" > $O 2>&1
TG_PR_CONCURRENT=0 timeout 600 python scripts/sweep_pr.py 28 "TG_PR_HUB=0;49152" >> $O 2>&1
cat $O
