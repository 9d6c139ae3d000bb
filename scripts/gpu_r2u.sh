#!/bin/bash
# L2 behaviour of the PageRank warp-class pull under cache-policy variants (ncu) + real round times
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum"
O=gpurun_out/r2u_policy.txt
: > $O
for V in "TG_PR_HOT=0" "TG_PR_HOT=4194304" "TG_PR_HOT=16777216" "TG_PR_L1=8" "TG_PR_HOT=16777216 TG_PR_NEXTPOL=2" "TG_PR_L1=1"; do
  env $V TG_PR_CONCURRENT=0 timeout 600 ncu --clock-control none --cache-control none $M -k regex:k_pull_warp -c 1 --csv --log-file /tmp/n.csv python scripts/prof_driver.py 28 pr > /dev/null 2>&1
  python - "$V" >> $O <<'PY'
import csv, sys
rows = list(csv.reader(open("/tmp/n.csv")))
hdr = None; out = []
for r in rows:
    if r and r[0] == "ID": hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r)); out.append(f"{d['Metric Name'].split('.')[0].replace('lts__t_sectors_srcunit_tex_op_read_lookup_','')}={d['Metric Value']}")
print(sys.argv[1], "warp-class ncu:", " ".join(out))
PY
done
timeout 900 python scripts/sweep_pr.py 28 "TG_PR_L1=0;8" >> $O 2>&1
cat $O
