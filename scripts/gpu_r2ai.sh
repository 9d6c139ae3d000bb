#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or direction" > gpurun_out/r2ai_tests.log 2>&1; tail -3 gpurun_out/r2ai_tests.log
timeout 1200 python scripts/sweep_env.py 28 "TG_PULL_HINTS=0;1;0;1" > gpurun_out/r2ai_hints.txt 2>&1
cat gpurun_out/r2ai_hints.txt
