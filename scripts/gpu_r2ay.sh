#!/bin/bash
# final validation on the head: smoke, full GPU suite, bench (as the driver runs them)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2ay_smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/r2ay_smoke.log
timeout 1800 python -m pytest tests -x -q -m gpu --durations=10 > gpurun_out/r2ay_pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2ay_pytest_gpu.log
timeout 900 python bench.py --out gpurun_out/r2ay_bench.json > gpurun_out/r2ay_bench.log 2>&1; echo "bench rc=$?" >> gpurun_out/r2ay_bench.log
tail -2 gpurun_out/r2ay_smoke.log; tail -3 gpurun_out/r2ay_pytest_gpu.log; tail -1 gpurun_out/r2ay_bench.log
python -c "import json; d=json.load(open('gpurun_out/r2ay_bench.json')); print(d['value'], d['ms_per_step'], d['per_algorithm_ms_per_step'], d['e2e']['value'], d['roofline']['frac'], d['clocks'])"
