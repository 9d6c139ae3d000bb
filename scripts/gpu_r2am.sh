#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants or direction or c1_ or partition_invariance" > gpurun_out/r2am_tests.log 2>&1; tail -3 gpurun_out/r2am_tests.log
timeout 1200 python scripts/sweep_env.py 28 "TG_BC_LEAN=0;1;0;1" > gpurun_out/r2am_bc_lean.txt 2>&1
cat gpurun_out/r2am_bc_lean.txt
