#!/bin/bash
# Cold-tail propagation blocking with chunked phase B (hub bins spread over many CTAs): parity + A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "cold_tail" > gpurun_out/r3an_tests.log 2>&1; tail -1 gpurun_out/r3an_tests.log
timeout 1500 python scripts/sweep_pr.py 28 "TG_PR_COLD=0;33554432;16777216;8388608;4194304" "TG_PR_COLD_KB=13;15" > gpurun_out/r3an_sweep.txt 2>&1
cat gpurun_out/r3an_sweep.txt
