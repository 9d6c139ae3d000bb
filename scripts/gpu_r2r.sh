#!/bin/bash
# TIMING PROBE: what each source range of the PageRank pull costs (gathers skipped, wrong results)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r2r_pr_skip.txt
echo "# TG_PR_L1=9: gathers of sources in [XLO, XHI) skipped (timing only)" > $O
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_L1=0" >> $O 2>&1
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_L1=9" "TG_PR_XLO=0" "TG_PR_XHI=0;49152;1048576;4194304" >> $O 2>&1
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_L1=9" "TG_PR_XLO=4194304;8388608;16777216;33554432" "TG_PR_XHI=4294967295" >> $O 2>&1
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_L1=9" "TG_PR_XLO=0" "TG_PR_XHI=4294967295" >> $O 2>&1
cat $O
