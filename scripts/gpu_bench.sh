#!/bin/bash
cd "$GRAFT_REPO_ROOT" 2>/dev/null || cd /root/repo
nproc > gpurun_out/host.txt; lscpu | grep "Model name" >> gpurun_out/host.txt; free -g >> gpurun_out/host.txt
timeout 900 python -m pytest tests -x -q -m gpu > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 900 python bench.py --scale 24 --steps 3 --warmup 2 --no-cpu-baseline --out gpurun_out/bench_s24.json > gpurun_out/bench_s24.log 2>&1; echo "rc=$?" >> gpurun_out/bench_s24.log
timeout 1500 python bench.py --scale 28 --steps 3 --warmup 2 --out gpurun_out/bench_s28.json > gpurun_out/bench_s28.log 2>&1; echo "rc=$?" >> gpurun_out/bench_s28.log
