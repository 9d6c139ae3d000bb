#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2v_tests.log 2>&1; tail -3 gpurun_out/r2v_tests.log
O=gpurun_out/r2v_pr_sweep.txt
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_PIPE=0;1;2;3" > $O 2>&1
TG_PR_CONCURRENT=0 timeout 900 python scripts/sweep_pr.py 28 "TG_PR_PIPE=0;1;2;3" >> $O 2>&1
cat $O
