#!/bin/bash
# DRAM bytes per random 4 B miss by allocation kind / fetch-granularity limit.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
./scripts/probes/fetch_probe > gpurun_out/r3m_fetch.txt 2>&1
M=dram__bytes_read.sum,lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric_op_read.sum,gpu__time_duration.sum
timeout 600 ncu --clock-control none --metrics $M -k regex:k_gather --csv --log-file gpurun_out/r3m_fetch_ncu.csv ./scripts/probes/fetch_probe > /dev/null 2>&1
cat gpurun_out/r3m_fetch.txt
