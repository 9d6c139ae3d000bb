#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for W in 0 1; do TG_BC_PULL_WALK=$W timeout 300 python scripts/time_algs.py 28 pullwalk=$W >> gpurun_out/bcpull.txt 2>&1; done
TG_TRACE=1 timeout 300 python scripts/trace_all.py 28 bc > gpurun_out/trace_bc.txt 2>&1
timeout 900 python -m pytest tests -x -q -m gpu -k "bc or direction or c2 or partition_invariance or golden or full" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -2 gpurun_out/pytest_gpu.log
