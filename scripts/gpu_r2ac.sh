#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "cold_tail" > gpurun_out/r2ac_tests.log 2>&1; tail -3 gpurun_out/r2ac_tests.log
O=gpurun_out/r2ac_pr_cold.txt
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_COLD=0;33554432;16777216;8388608;4194304" "TG_PR_COLD_KB=15;14" > $O 2>&1
cat $O
