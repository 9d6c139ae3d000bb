#!/bin/bash
# PageRank: rows of out-degree 0 skip the next contribution (TG_PR_NZSKIP) -- parity + A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r3w_tests.log 2>&1; tail -2 gpurun_out/r3w_tests.log
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_NZSKIP=0;1;0;1;0;1" > gpurun_out/r3w_sweep.txt 2>&1
cat gpurun_out/r3w_sweep.txt
