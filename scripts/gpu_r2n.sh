#!/bin/bash
# per-kernel durations of one PageRank round with / without the hub split (ncu launch list)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,lts__t_sector_hit_rate.pct,l1tex__data_pipe_lsu_wavefronts_mem_shared.sum,smsp__inst_executed.sum"
for K in 0 49152; do
TG_PR_HUB=$K TG_PR_CONCURRENT=0 timeout 900 ncu --clock-control none --cache-control none $M -k regex:k_pull --csv --log-file gpurun_out/r2n_hub$K.csv python scripts/prof_driver.py 28 pr > gpurun_out/r2n_hub$K.log 2>&1
done
python - <<'PY'
import csv
for K in (0, 49152):
    rows = list(csv.reader(open(f"gpurun_out/r2n_hub{K}.csv")))
    hdr = None
    for r in rows:
        if r and r[0] == "ID": hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            print(K, d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"])
PY
