#!/bin/bash
# BC lazy zeroing of sigma / dsum (TG_BC_LAZYZERO): parity (several sources per call, repeated calls) + A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py tests/test_multiproc.py -m gpu -x -q > gpurun_out/r3ad_tests.log 2>&1; tail -1 gpurun_out/r3ad_tests.log
timeout 900 python scripts/sweep_env.py 28 "TG_BC_LAZYZERO=0;1;0;1" > gpurun_out/r3ad_sweep.txt 2>&1
cat gpurun_out/r3ad_sweep.txt
