#!/bin/bash
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
for X in 0 4294967295; do
TG_PR_L1=9 TG_PR_XLO=0 TG_PR_XHI=$X TG_PR_CONCURRENT=0 timeout 600 ncu --clock-control none --cache-control none --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active -k regex:k_pull -c 3 --csv --log-file /tmp/sk$X.csv python scripts/prof_driver.py 28 pr > /dev/null 2>&1
python - $X <<'PY'
import csv, sys
rows = list(csv.reader(open(f"/tmp/sk{sys.argv[1]}.csv")))
hdr = None
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); print("skip_hi", sys.argv[1], d["Kernel Name"][:28], d["Metric Name"], d["Metric Value"])
PY
done
