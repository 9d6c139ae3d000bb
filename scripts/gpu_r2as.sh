#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2as_tests.log 2>&1; tail -3 gpurun_out/r2as_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_F32DIV=0;1;0;1" > gpurun_out/r2as.txt 2>&1
cat gpurun_out/r2as.txt
