#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
for U in 4 8; do TG_UNROLL=$U timeout 300 python scripts/time_algs.py 28 U=$U >> gpurun_out/unroll.txt 2>&1; done
timeout 300 python scripts/time_algs.py 28 default >> gpurun_out/unroll.txt 2>&1
timeout 1500 python -m pytest tests -x -q -m gpu --durations=8 > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
tail -14 gpurun_out/pytest_gpu.log
