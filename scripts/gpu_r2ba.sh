#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or hub_split or ghost" > gpurun_out/r2ba_tests.log 2>&1; tail -3 gpurun_out/r2ba_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_HALF=;4;8;16;;8" > gpurun_out/r2ba.txt 2>&1
cat gpurun_out/r2ba.txt
