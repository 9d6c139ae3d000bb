#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2x_tests.log 2>&1; tail -3 gpurun_out/r2x_tests.log
O=gpurun_out/r2x_sssp_hot.txt
timeout 1200 python scripts/sweep_env.py 28 "TG_SSSP_HOT=0;4194304;16777216;33554432;268435456" > $O 2>&1
cat $O
