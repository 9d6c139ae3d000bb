#!/bin/bash
# Re-tune sweep of schedule knobs on the final library (results are schedule-invariant).
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python scripts/sweep_env.py 28 "TG_SSSP_DELTA=1;2;4" "TG_SSSP_HUB_DEG=64;128;256" > gpurun_out/r3v_sssp.txt 2>&1
timeout 600 python scripts/sweep_env.py 28 "TG_BC_PRIV=256;512;1024;2048" > gpurun_out/r3v_bc.txt 2>&1
timeout 600 python scripts/sweep_env.py 28 "TG_BU_ALPHA=8;14;24" "TG_BC_ALPHA=1;2;4" > gpurun_out/r3v_dir.txt 2>&1
cat gpurun_out/r3v_sssp.txt gpurun_out/r3v_bc.txt gpurun_out/r3v_dir.txt
