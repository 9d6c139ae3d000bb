#!/bin/bash
# Binned collection (TG_COLLECT=3): parity, permutation cost, e2e bench A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
TG_COLLECT=3 timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q > gpurun_out/r3o_tests.log 2>&1; tail -3 gpurun_out/r3o_tests.log
timeout 600 python scripts/time_collect_dev.py 28 > gpurun_out/r3o_collect.txt 2>&1
cat gpurun_out/r3o_collect.txt
timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3o_bench_mode2.json 2>/dev/null
TG_COLLECT=3 timeout 900 python bench.py --no-cpu-baseline > gpurun_out/r3o_bench_mode3.json 2>/dev/null
for f in gpurun_out/r3o_bench_mode2.json gpurun_out/r3o_bench_mode3.json; do python -c "
import json,sys; d=json.loads(open('$f').read().strip().splitlines()[-1]); print('$f', 'value', round(d['value'],1), 'e2e', round(d['e2e']['value'],1), 'clk', d['clocks']['sm_mhz'])"; done
