#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or golden or c1_" > gpurun_out/r2an_tests.log 2>&1; tail -3 gpurun_out/r2an_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_POLPARAM=0;1;0;1" > gpurun_out/r2an_polparam.txt 2>&1
cat gpurun_out/r2an_polparam.txt
