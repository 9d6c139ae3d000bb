#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1200 python scripts/sweep_env.py 28 "TG_SSSP_CLASS_SPARSE=0;16;64;256;0" > gpurun_out/r2at.txt 2>&1
cat gpurun_out/r2at.txt
TG_SSSP_CLASS_SPARSE=64 TG_TRACE=1 timeout 600 python scripts/trace_all.py 28 sssp > gpurun_out/r2at_trace.txt 2>&1; grep "step=" gpurun_out/r2at_trace.txt | head -12
