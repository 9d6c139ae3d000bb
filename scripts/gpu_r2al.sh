#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants and PRED" > gpurun_out/r2al_tests.log 2>&1; tail -3 gpurun_out/r2al_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_PRED=0,0,0;-8,-8,-4;-108,-108,-4;-8,-108,-4;-108,-8,-4;-16,-8,-4;-16,-108,-4;-8,-8,-4;-108,-108,-4" > gpurun_out/r2al_pred.txt 2>&1
cat gpurun_out/r2al_pred.txt
