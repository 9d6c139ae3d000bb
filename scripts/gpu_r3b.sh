#!/bin/bash
# Carveout A/B (TG_CARVEOUT) of the PageRank class pulls and the frontier walkers, RMAT-28.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/sweep_env.py 28 "TG_CARVEOUT=;0;100;50;0" > gpurun_out/r3b_sweep.txt 2>&1
cat gpurun_out/r3b_sweep.txt
