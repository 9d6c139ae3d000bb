#!/bin/bash
# C4 full oracle at RMAT-28 incl. the opt-in connected-components union-find parity
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
free -g > gpurun_out/r2aq_c4_cc.log; nproc >> gpurun_out/r2aq_c4_cc.log
TG_C4_CC=1 timeout 3300 python -m pytest tests/test_gpu_fullscale.py -m gpu -q -s -k full_oracle --durations=3 >> gpurun_out/r2aq_c4_cc.log 2>&1
echo "rc=$?" >> gpurun_out/r2aq_c4_cc.log
tail -8 gpurun_out/r2aq_c4_cc.log
