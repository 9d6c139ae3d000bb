#!/bin/bash
# L2 sector accounting of random 4 B gathers (l2_probe2 k_hash<4>): sectors per gather by region size,
# split by source unit (tex vs fabric) -- are far-die lines looked up twice?
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,lts__t_sectors_srcunit_ltcfabric_op_read.sum,lts__t_sectors_op_read.sum,dram__bytes_read.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,gpu__time_duration.sum
timeout 900 ncu --clock-control none --metrics $M -k regex:"k_hash<4>" --csv --log-file gpurun_out/r3k_probe.csv ./scripts/probes/l2_probe2 > gpurun_out/r3k_probe.log 2>&1
M2=lts__t_sectors_srcunit_tex_op_read.sum,lts__t_sectors_srcunit_ltcfabric_op_read.sum,lts__t_sectors_op_read.sum,lts__t_sectors_op_atom.sum,lts__t_sectors_op_red.sum,lts__t_sectors_op_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,dram__bytes_read.sum,gpu__time_duration.sum
timeout 900 ncu --clock-control none --metrics $M2 -k regex:k_pull --csv --log-file gpurun_out/r3k_pr.csv python scripts/prof_driver.py 28 pr > gpurun_out/r3k_pr.log 2>&1
ls -la gpurun_out | tail -5
