#!/bin/bash
cd "$(dirname "$0")/.."
python scripts/time_e2e_async.py 28 > gpurun_out/r2j_e2e_async.txt 2>&1
cat gpurun_out/r2j_e2e_async.txt
python bench.py --steps 10 --warmup 3 --out gpurun_out/r2j_bench.json > gpurun_out/r2j_bench.log 2>&1
tail -c 400 gpurun_out/r2j_bench.log
python -m pytest tests/test_gpu_parity.py tests/test_multiproc.py -m gpu -q -x > gpurun_out/r2j_tests.log 2>&1; tail -2 gpurun_out/r2j_tests.log
