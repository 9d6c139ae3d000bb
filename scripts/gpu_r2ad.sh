#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "in_csr_only or ghost_pull or c1_" > gpurun_out/r2ad_tests.log 2>&1; tail -3 gpurun_out/r2ad_tests.log
free -g > gpurun_out/r2ad_rmat30_pr.log; nproc >> gpurun_out/r2ad_rmat30_pr.log
TG_RMAT30=1 timeout 2700 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k rmat30_pagerank --durations=3 >> gpurun_out/r2ad_rmat30_pr.log 2>&1
echo "rc=$?" >> gpurun_out/r2ad_rmat30_pr.log
tail -12 gpurun_out/r2ad_rmat30_pr.log
