#!/bin/bash
# round-2 evidence: per-superstep traces, ncu launch list of the bench, --set full of the hot kernels
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 600 python scripts/trace_all.py 28 sssp,bc > gpurun_out/r2w_trace_s28.txt 2>&1
S=28 bash scripts/gpu_ncu.sh
ls gpurun_out/*.ncu-rep
