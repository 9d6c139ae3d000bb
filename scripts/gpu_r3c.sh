#!/bin/bash
# L2 persisting-limit A/B (TG_L2_PERSIST) + DRAM bytes of the PageRank pulls vs the hot prefix.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "
from cuda.bindings import runtime as rt
print('persist default', rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitPersistingL2CacheSize), 'max', rt.cudaDeviceGetAttribute(rt.cudaDeviceAttr.cudaDevAttrMaxPersistingL2CacheSize, 0))
" > gpurun_out/r3c_sweep.txt 2>&1
timeout 900 python scripts/sweep_pr.py 28 "TG_L2_PERSIST=;33554432;67108864;-1;0" >> gpurun_out/r3c_sweep.txt 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_tex_op_read.sum
for h in 4194304 8388608 16777216; do
  TG_PR_HOT=$h timeout 600 ncu --clock-control none --metrics $M -k regex:k_pull --csv --log-file gpurun_out/r3c_ncu_hot$h.csv python scripts/prof_driver.py 28 pr > /dev/null 2>&1
done
TG_L2_PERSIST=-1 timeout 600 ncu --clock-control none --metrics $M -k regex:k_pull --csv --log-file gpurun_out/r3c_ncu_persist.csv python scripts/prof_driver.py 28 pr > /dev/null 2>&1
cat gpurun_out/r3c_sweep.txt
