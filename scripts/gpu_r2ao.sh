#!/bin/bash
# bench + ncu evidence refresh after the lean PageRank batches
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/r2ao_bench.json > gpurun_out/r2ao_bench.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/r2ao_bench.json')); print(d['value'], d['per_algorithm_ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['roofline']['gather_bound'])"
S=28 bash scripts/gpu_ncu.sh > /dev/null 2>&1
ls gpurun_out/*.ncu-rep
