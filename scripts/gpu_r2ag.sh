#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2ag_tests.log 2>&1; tail -3 gpurun_out/r2ag_tests.log
timeout 1200 python scripts/sweep_env.py 28 "TG_BC_PRIV_MODE=0;1;2" "TG_BC_PRIV=512;2048;8192" > gpurun_out/r2ag_bc_priv.txt 2>&1
cat gpurun_out/r2ag_bc_priv.txt
