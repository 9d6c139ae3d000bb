#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r2aw.txt; : > $O
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_HOT=8388608;16777216;25165824;33554432" "TG_PR_CONCURRENT=1;0" >> $O 2>&1
timeout 900 python scripts/sweep_env.py 28 "TG_BC_PRIV=256;512;1024;2048" >> $O 2>&1
cat $O
