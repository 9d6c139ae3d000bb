#!/bin/bash
# PageRank: next-contribution L2 policy x hot prefix; shared-memory hub replica at 2 CTAs/SM
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r2l_pr_sweep.txt
timeout 600 python scripts/sweep_pr.py 28 "TG_PR_NEXTPOL=0;1;2" "TG_PR_HOT=16777216;25165824;33554432" > $O 2>&1
timeout 600 python scripts/sweep_pr.py 28 "TG_PR_NEXTPOL=0;2" "TG_PR_REP=0;8192;16384;24576" "TG_PR_REP_CLASSES=2;6" >> $O 2>&1
TG_PR_REP_CTAS=1 timeout 300 python scripts/sweep_pr.py 28 "TG_PR_NEXTPOL=2" "TG_PR_REP=32768;49152" >> $O 2>&1
cat $O
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2l_tests.log 2>&1; tail -3 gpurun_out/r2l_tests.log
