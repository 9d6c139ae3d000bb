#!/bin/bash
# True (application-replay, warm-cache) DRAM bytes / L2 hit rates of the PageRank class pulls,
# second round of a 2-round run (kernel-replay ncu restores memory between passes and distorts L2 state)
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
M="--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,lts__t_sectors_srcunit_tex_op_read_lookup_hit.sum,lts__t_sectors_srcunit_tex_op_read_lookup_miss.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,smsp__inst_executed.sum"
cat > /tmp/pr2.py <<'PY'
import sys; sys.path.insert(0, ".")
import paper_1312_3018_b200 as tg
eng = tg.Engine.rmat(28)
print(eng.pagerank(2)[1])
PY
for C in 1 0; do
TG_PR_CONCURRENT=$C timeout 900 ncu --replay-mode application --clock-control none --cache-control none $M -k regex:k_pull -s 3 -c 3 --csv --log-file gpurun_out/r2t_app_c$C.csv python /tmp/pr2.py > gpurun_out/r2t_app_c$C.log 2>&1
done
python - <<'PY'
import csv
for C in (1, 0):
    rows = list(csv.reader(open(f"gpurun_out/r2t_app_c{C}.csv")))
    hdr = None
    for r in rows:
        if r and r[0] == "ID": hdr = r; continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            print(C, d["Kernel Name"][:30], d["Metric Name"], d["Metric Value"])
PY
