#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_cc.py -m gpu -q -x > gpurun_out/r2ar_tests.log 2>&1; tail -3 gpurun_out/r2ar_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --out gpurun_out/r2ar_bench.json > gpurun_out/r2ar_bench.log 2>&1
python -c "import json; d=json.load(open('gpurun_out/r2ar_bench.json')); print(d['value'], d['per_algorithm_ms_per_step'], d['e2e']['value'])"
