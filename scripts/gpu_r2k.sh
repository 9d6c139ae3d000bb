#!/bin/bash
# round-2 re-entry check: probe v2, hub coverage, bench, GPU parity suite (no full-scale file)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/r2k_gpu.txt 2>&1
timeout 300 scripts/probes/l2_probe2 > gpurun_out/r2k_l2_probe2.txt 2>&1
timeout 300 python scripts/pr_coverage.py 28 > gpurun_out/r2k_pr_coverage.txt 2>&1
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/r2k_bench.json > gpurun_out/r2k_bench.log 2>&1
tail -c 600 gpurun_out/r2k_bench.log
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_multiproc.py tests/test_gpu_cc.py -m gpu -q -x > gpurun_out/r2k_tests.log 2>&1; tail -3 gpurun_out/r2k_tests.log
cat gpurun_out/r2k_l2_probe2.txt gpurun_out/r2k_pr_coverage.txt
