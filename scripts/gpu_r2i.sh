#!/bin/bash
cd "$(dirname "$0")/.."
python scripts/time_e2e_async.py 28 > gpurun_out/r2i_e2e_async.txt 2>&1
python -m pytest tests/test_multiproc.py -m gpu -q -x > gpurun_out/r2i_multiproc.log 2>&1
python scripts/time_exchange.py 26 8 > gpurun_out/r2i_partitions_s26_P8.txt 2>&1
cat gpurun_out/r2i_e2e_async.txt; tail -3 gpurun_out/r2i_multiproc.log; cat gpurun_out/r2i_partitions_s26_P8.txt
