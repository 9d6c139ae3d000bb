#!/bin/bash
# PageRank: non-final rounds do not pull the sinks' rows (TG_PR_SINKSKIP) -- parity + A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r3z_tests.log 2>&1; tail -2 gpurun_out/r3z_tests.log
timeout 1200 python scripts/sweep_pr.py 28 "TG_PR_SINKSKIP=0;1;0;1;0;1" > gpurun_out/r3z_sweep.txt 2>&1
cat gpurun_out/r3z_sweep.txt
