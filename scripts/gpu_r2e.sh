#!/bin/bash
# round-2 experiment batch: PageRank L1 placement sweep, SSSP dense-step A/B, sanitizers
cd "$(dirname "$0")/.."
python scripts/sweep_pr.py 28 "TG_PR_L1=0;1;2" > gpurun_out/r2_pr_l1.txt 2>&1
python scripts/sweep_pr.py 28 "TG_PR_L1=3" "TG_PR_L1HOT=4096;16384;65536" >> gpurun_out/r2_pr_l1.txt 2>&1
python scripts/sweep_sssp_dense.py 28 > gpurun_out/r2_sssp_dense.txt 2>&1
for tool in memcheck racecheck synccheck; do
  timeout 900 compute-sanitizer --tool $tool --print-limit 50 python scripts/sanitize_c1.py > gpurun_out/r2_sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" >> gpurun_out/r2_sanitize_$tool.txt
done
tail -3 gpurun_out/r2_*.txt
