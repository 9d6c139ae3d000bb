#!/bin/bash
# round-2 batch: BC hub-pull sweep, P-partition timings with direction optimization, BFS top-only reference
cd "$(dirname "$0")/.."
python scripts/sweep_env.py 28 "TG_BC_HUBPULL=0;512;2048;8192;32768" > gpurun_out/r2_bc_hubpull.txt 2>&1
for P in 1 2 4 8; do python scripts/time_exchange.py 26 $P; done > gpurun_out/r2_partitions_s26.txt 2>&1
for P in 1 8; do TG_DIRECTION=top python scripts/time_exchange.py 26 $P; done > gpurun_out/r2_partitions_s26_topdown.txt 2>&1
tail -20 gpurun_out/r2_bc_hubpull.txt gpurun_out/r2_partitions_s26*.txt
