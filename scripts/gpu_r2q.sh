#!/bin/bash
# ncu metrics of the die-split PageRank kernels vs the class pulls (one round, RMAT-28)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active"
TG_PR_SPLIT=1 timeout 900 ncu --clock-control none --cache-control none $M -k regex:"k_pr_split|k_split|k_pull" --csv --log-file gpurun_out/r2q_split.csv python scripts/prof_driver.py 28 pr > gpurun_out/r2q_split.log 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open("gpurun_out/r2q_split.csv")))
hdr = None
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        print(d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"])
PY
