#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2ak_tests.log 2>&1; tail -3 gpurun_out/r2ak_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_PRED=0,0,0;0,4,0;0,6,0;0,8,0;0,0,2;0,0,4;4,0,0;4,8,4;2,6,2" > gpurun_out/r2ak_pred.txt 2>&1
cat gpurun_out/r2ak_pred.txt
