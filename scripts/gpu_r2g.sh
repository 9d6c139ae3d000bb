#!/bin/bash
# round-2 batch g: new parity tests, traces at P=1 / P=8 (RMAT-26), bench with async e2e, PR seg A/B
cd "$(dirname "$0")/.."
python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "variants or async or direction" > gpurun_out/r2g_tests.log 2>&1
tail -3 gpurun_out/r2g_tests.log
for P in 1 8; do python scripts/trace_all.py 26 bfs,sssp,bc $P > gpurun_out/r2g_trace_s26_P$P.txt 2>&1; done
python scripts/sweep_pr.py 28 "TG_PR_SEG=0;1" > gpurun_out/r2g_pr_seg.txt 2>&1
python bench.py --steps 10 --warmup 3 --out gpurun_out/r2g_bench.json > gpurun_out/r2g_bench.log 2>&1
tail -c 600 gpurun_out/r2g_bench.log; cat gpurun_out/r2g_pr_seg.txt
