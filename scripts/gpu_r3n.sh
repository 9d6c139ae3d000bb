#!/bin/bash
# 16-bit SSSP distances (TG_SSSP_D16): parity with the mode forced on, then the RMAT-28 A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TG_SSSP_D16=1 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r3n_tests.log 2>&1; tail -3 gpurun_out/r3n_tests.log
timeout 900 python scripts/sweep_env.py 28 "TG_SSSP_D16=0;1;0;1" > gpurun_out/r3n_sweep.txt 2>&1
cat gpurun_out/r3n_sweep.txt
