#!/bin/bash
# Per-partition streams (each_part) for BFS: multi-partition parity, then RMAT-26 P = 1/2/4/8 timings, streams on vs off.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fuzz.py -m gpu -x -q -k "not c2 and not c3" > gpurun_out/r3g_tests.log 2>&1; tail -3 gpurun_out/r3g_tests.log
for P in 1 2 4 8; do
  for ps in 0 1; do
    TG_PART_STREAMS=$ps timeout 600 python scripts/time_exchange.py 26 $P 2>&1 | sed "s/^/streams=$ps /" >> gpurun_out/r3g_times.txt
  done
done
cat gpurun_out/r3g_times.txt
