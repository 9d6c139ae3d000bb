#!/bin/bash
# round-2 batch h: bench (async e2e), then the whole GPU suite with its wall time
cd "$(dirname "$0")/.."
python bench.py --steps 10 --warmup 3 --out gpurun_out/r2h_bench.json > gpurun_out/r2h_bench.log 2>&1
tail -c 300 gpurun_out/r2h_bench.log
start=$(date +%s)
python -m pytest tests -m gpu -q > gpurun_out/r2h_pytest_gpu.log 2>&1
echo "pytest -m gpu rc=$? wall=$(( $(date +%s) - start )) s" >> gpurun_out/r2h_pytest_gpu.log
tail -5 gpurun_out/r2h_pytest_gpu.log
