#!/bin/bash
# L2 fetch-granularity A/B (TG_L2_FETCH) on RMAT-28 + ncu DRAM bytes of the
# PageRank pulls under each, then the full GPU suite on this head.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
python -c "
from cuda.bindings import runtime as rt
print('default MaxL2FetchGranularity', rt.cudaDeviceGetLimit(rt.cudaLimit.cudaLimitMaxL2FetchGranularity))
" > gpurun_out/r3a_default.txt 2>&1
timeout 900 python scripts/sweep_env.py 28 "TG_L2_FETCH=;32;64;128;32" > gpurun_out/r3a_sweep.txt 2>&1
for g in 32 128; do
  TG_L2_FETCH=$g timeout 600 ncu --clock-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum -k regex:"k_pull|SsspOp" --csv --log-file gpurun_out/r3a_ncu_$g.csv python scripts/prof_driver.py 28 pr,sssp > gpurun_out/r3a_ncu_$g.log 2>&1
done
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r3a_pytest_gpu.log 2>&1
tail -3 gpurun_out/r3a_pytest_gpu.log
cat gpurun_out/r3a_default.txt gpurun_out/r3a_sweep.txt
