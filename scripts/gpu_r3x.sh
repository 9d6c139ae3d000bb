#!/bin/bash
# PageRank skeleton trims: rank stored by the last round only (TG_PR_RANKLAST), thread class skips
# offsets of rows without in-edges (TG_PR_INNZ) -- parity + A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r3x_tests.log 2>&1; tail -2 gpurun_out/r3x_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_RANKLAST=0;1" "TG_PR_INNZ=0;1" > gpurun_out/r3x_sweep.txt 2>&1
timeout 600 python scripts/sweep_pr.py 28 "TG_PR_RANKLAST=0;1" "TG_PR_INNZ=0;1" >> gpurun_out/r3x_sweep.txt 2>&1
cat gpurun_out/r3x_sweep.txt
