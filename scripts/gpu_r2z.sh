#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "variants" > gpurun_out/r2z_tests.log 2>&1; tail -3 gpurun_out/r2z_tests.log
O=gpurun_out/r2z_sssp_cls.txt
timeout 1200 python scripts/sweep_env.py 28 "TG_SSSP_CLASS_DIV=0;4;16;64" > $O 2>&1
cat $O
TG_SSSP_CLASS_DIV=16 TG_TRACE=1 timeout 600 python scripts/trace_all.py 28 sssp > gpurun_out/r2z_trace.txt 2>&1; grep "step=[3-8] " gpurun_out/r2z_trace.txt
