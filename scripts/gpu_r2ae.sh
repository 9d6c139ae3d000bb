#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2ae_tests.log 2>&1; tail -3 gpurun_out/r2ae_tests.log
timeout 1200 python scripts/ab_build_env.py 28 "TG_ORDER_LOCAL=0;1" > gpurun_out/r2ae_order.txt 2>&1
cat gpurun_out/r2ae_order.txt
