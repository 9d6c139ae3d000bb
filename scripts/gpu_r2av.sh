#!/bin/bash
# walker unroll re-sweep after the window pre-scan (TG_UNROLL overrides every op; fresh process each)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
O=gpurun_out/r2av_unroll.txt; : > $O
for U in default 2 3 4 8; do
  if [ $U = default ]; then timeout 600 python scripts/sweep_env.py 28 "TG_X=$U" >> $O 2>&1
  else TG_UNROLL=$U timeout 600 python scripts/sweep_env.py 28 "TG_X=U$U" >> $O 2>&1; fi
done
cat $O
