#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "short_row or variants" > gpurun_out/r2s_tests.log 2>&1; tail -3 gpurun_out/r2s_tests.log
O=gpurun_out/r2s_pr_sweep.txt
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_GROUP=0;1" > $O 2>&1
TG_PR_CONCURRENT=0 timeout 900 python scripts/sweep_pr.py 28 "TG_PR_GROUP=0;1" >> $O 2>&1
cat $O
