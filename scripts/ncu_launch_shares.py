"""profiles/<round>_ncu_launch_shares.csv from an ncu --csv launch list
(scripts/gpu_ncu.sh): per-kernel share of the algorithm-kernel time (build
launches excluded) and DRAM bytes, to compare with the bench ledger's shares."""
import collections
import csv
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
src = sys.argv[1] if len(sys.argv) > 1 else os.path.join(ROOT, "gpurun_out", "launches.csv")
rnd = sys.argv[2] if len(sys.argv) > 2 else "r01"
rows = list(csv.reader(open(src)))
hi = next(i for i, r in enumerate(rows) if r and r[0] == "ID")
hdr = rows[hi]
ki, mi, vi, ui = (hdr.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit"))
TS = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}
BS = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launch, by_id = [], {}
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    if r[0] not in by_id:
        by_id[r[0]] = [r[ki].split("(")[0], 0.0, 0.0]
        launch.append(by_id[r[0]])
    v = float(r[vi].replace(",", ""))
    if r[mi] == "gpu__time_duration.sum":
        by_id[r[0]][1] = v * TS[r[ui]]
    elif r[mi].startswith("dram__bytes"):
        by_id[r[0]][2] += v * BS[r[ui]]
ALG = ("k_advance", "k_seed", "k_pr_init", "k_warp_expand", "k_bc_seed")
first = next(i for i, l in enumerate(launch) if any(a in l[0] for a in ALG))
build, alg = launch[:first], launch[first:]
t, n, b = collections.defaultdict(float), collections.Counter(), collections.defaultdict(float)
for k, ms, by in alg:
    t[k] += ms
    n[k] += 1
    b[k] += by
tot = sum(t.values())
out = [f"# ncu launch list ({os.path.basename(src)}), --clock-control none, serialised cold-cache replays.",
       f"# {len(build)} build launches (untimed engine construction) excluded; {len(alg)} algorithm "
       f"launches (warm-up + timed step) = {tot:.2f} ms.",
       "# share = fraction of the algorithm-kernel time; compare with bench.py's share_of_kernel_time.",
       "kernel,launches,ms,share,dram_GB"]
for k, v in sorted(t.items(), key=lambda x: -x[1]):
    out.append(f"{k},{n[k]},{v:.3f},{v / tot:.4f},{b[k] / 1e9:.2f}")
pr = sum(v for k, v in t.items() if "k_pull" in k)
out.append(f"# PageRank pull kernels (k_pull_*) together: share {pr / tot:.4f}")
open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_launch_shares.csv"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:14] + out[-1:]))
