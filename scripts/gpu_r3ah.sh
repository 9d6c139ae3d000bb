#!/bin/bash
# SSSP: sinks are not activated when their distance drops (TG_SSSP_SINKS=1 restores) -- parity + A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_multiproc.py -m gpu -x -q > gpurun_out/r3ah_tests.log 2>&1; tail -1 gpurun_out/r3ah_tests.log
timeout 900 python scripts/sweep_env.py 28 "TG_SSSP_SINKS=1;0;1;0" > gpurun_out/r3ah_sweep.txt 2>&1
cat gpurun_out/r3ah_sweep.txt
