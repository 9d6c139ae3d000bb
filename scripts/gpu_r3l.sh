#!/bin/bash
# Load-flavor gather probe: time + L1 / L2 sector accounting per flavor.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
./scripts/probes/gather_flavors > gpurun_out/r3l_flavors.txt 2>&1
M=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_ltcfabric_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sector_hit_rate.pct,dram__bytes_read.sum,gpu__time_duration.sum
timeout 900 ncu --clock-control none --metrics $M -k regex:k_gather --csv --log-file gpurun_out/r3l_flavors_ncu.csv ./scripts/probes/gather_flavors > /dev/null 2>&1
cat gpurun_out/r3l_flavors.txt
