"""Summarise ncu reports in gpurun_out/ into profiles/<round>_ncu_summary.md and
profiles/ncu_traffic.json (per-launch DRAM bytes of each ledger kernel)."""
import csv
import io
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
OUT = os.path.join(ROOT, "gpurun_out")
rnd = sys.argv[1] if len(sys.argv) > 1 else "r01"
try:
    PEAK = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
except (OSError, KeyError, ValueError):
    PEAK = 6537.3
WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "smsp__inst_executed.sum",
        # sector efficiency: useful bytes per 32-byte sector
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio",
        "smsp__sass_average_data_bytes_per_sector_mem_global_op_st.ratio"]
STALLS = ["long_scoreboard", "barrier", "wait", "short_scoreboard", "lg_throttle", "mio_throttle",
          "math_pipe_throttle", "not_selected", "selected", "branch_resolving", "membar", "drain"]
LEDGER = {"prof_pr": "pr_pull", "prof_bfs": "bfs_expand", "prof_sssp": "sssp_expand",
          "prof_bcf": "bc_fwd_expand", "prof_bcb": "bc_bwd_expand"}


def to_bytes(v, unit):
    f = float(v)
    return f * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(unit, 1)


lines = [f"# ncu summary ({rnd})", "",
         "`ncu --set full --clock-control none` captures (cold-cache, serialised replays;",
         "compare shares, not absolutes).  Source: scripts/gpu_ncu.sh, scripts/prof_driver.py.", ""]
traffic = {}
for rep in sorted(f for f in os.listdir(OUT) if f.endswith(".ncu-rep")):
    name = rep[:-8]
    raw = subprocess.run(["ncu", "-i", os.path.join(OUT, rep), "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    if len(rows) < 3:
        continue
    hdr, units = rows[0], rows[1]
    lines.append(f"## {name}")
    lines.append("")
    per_launch = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        kname = d.get("Kernel Name", "?")[:70]
        lines.append(f"### `{kname}`")
        for w in WANT:
            if w in d:
                lines.append(f"- {w}: {d[w]} {u.get(w, '')}")
        st = []
        for s in STALLS:
            k = f"smsp__pcsamp_warps_issue_stalled_{s}"
            if k in d and d[k] not in ("", "0"):
                st.append((int(float(d[k])), s))
        st.sort(reverse=True)
        lines.append("- top stall samples: " + ", ".join(f"{s}={n}" for n, s in st[:6]))
        try:  # derived: achieved DRAM bandwidth and load sector efficiency
            t_ms = float(d["gpu__time_duration.sum"]) * {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3,
                                                           "usecond": 1e-3}.get(
                u["gpu__time_duration.sum"], 1.0)
            by = (to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) +
                  to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
            gbs = by / (t_ms * 1e-3) / 1e9
            eff = float(d["smsp__sass_average_data_bytes_per_sector_mem_global_op_ld.ratio"]) / 32
            lines.append(f"- derived: DRAM {gbs:.0f} GB/s = {gbs / PEAK:.2f} of {PEAK:.0f} GB/s "
                         f"(cold, serialised replay); load sector efficiency {eff:.2f}")
        except (KeyError, ValueError, ZeroDivisionError):
            pass
        lines.append("")
        try:
            per_launch.append(to_bytes(d["dram__bytes_read.sum"], u["dram__bytes_read.sum"]) +
                              to_bytes(d["dram__bytes_write.sum"], u["dram__bytes_write.sum"]))
        except (KeyError, ValueError):
            pass
    if name in LEDGER and per_launch:
        # pr_pull's ledger unit is one round = the three class kernels together
        traffic[LEDGER[name]] = sum(per_launch) if name == "prof_pr" else max(per_launch)
os.makedirs(os.path.join(ROOT, "profiles"), exist_ok=True)
open(os.path.join(ROOT, "profiles", f"{rnd}_ncu_summary.md"), "w").write("\n".join(lines) + "\n")
json.dump(traffic, open(os.path.join(ROOT, "profiles", "ncu_traffic.json"), "w"), indent=1)
print("\n".join(lines[:80]))
print(traffic)
