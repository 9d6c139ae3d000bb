#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/r2y_bench.json > gpurun_out/r2y_bench.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/r2y_bench.json')); print(d['value'], d['per_algorithm_ms_per_step'], d['e2e']['value'])"
timeout 600 python scripts/trace_all.py 28 sssp > gpurun_out/r2y_trace.txt 2>&1; head -3 gpurun_out/r2y_trace.txt
timeout 600 python scripts/sweep_env.py 28 "TG_SSSP_HOT=0" 2>&1 | tail -1
