#!/usr/bin/env python
"""bench.py -- the TOTEM BSP superstep hot path on B200 (BASELINE.json metric).

One "step" = one pass of every hot-path row of SURVEY.md 8(a) over the
resident RMAT graph: BFS from source j, Bellman-Ford SSSP from source j,
PageRank (5 Jacobi rounds, the paper's Fig. 16 protocol) and Brandes BC from
source j.  The workload at N=1 is RMAT-28 (edge factor 16, 2^32 edges), the
configuration BASELINE.json's metric is quoted on; it fits one B200.

value  = traversed edges of the whole step (the paper's TEPS numerators,
         PAPER.md:336: BFS/SSSP sum of reached out-degrees, BC 2x that,
         PageRank |E| per round) / device time of the step, in GTEPS,
         outputs written to device memory.  Device time = sum of the CUDA-event
         intervals the library records on its own stream around each algorithm
         (state init .. final vote), bracketed by barrier + synchronize.
e2e    = same metric through the same C-ABI calls with HOST output buffers
         (pinned), device->host copies of every result inside the timed region.
roofline = the dominant kernel from the library's CUDA-event kernel ledger.
cpu_baseline = the CPU oracle (single thread) on a bounded RMAT-22 sample.

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "BFS/SSSP/BC GTEPS and PageRank edges/s/iter, RMAT-28 at 1/2/4/8 B200"
UNIT = "GTEPS"
PR_ITERS = 5


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="tgraph", choices=["tgraph", "reference"])
    ap.add_argument("--scale", type=int, default=28)
    ap.add_argument("--cpu-scale", type=int, default=22, help="RMAT scale of the oracle sample")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--out", default=None, help="also write the JSON line to this file")
    return ap.parse_args()


# ----------------------------------------------------------------- helpers
class ClockSampler:
    """nvidia-smi sampling during the timed region (B200_PROFILING.md clocks line)."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.proc, self.lines = index, None, []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], 0.0, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = max(mx, float(f[2]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def gather_probe_ceiling():
    """Best rate (gathers/s) of PageRank's own access pattern -- a coalesced
    4-byte index stream + dependent random 4-byte gathers from an L2-resident
    region -- in the committed round-2 probe table (scripts/probes/l2_probe2.cu;
    its hashed-index columns reach ~290 G/s, the L1TEX one-line-per-clock
    rate).  The round-1 probe's 230 G/s was bounded by its own index arithmetic."""
    path = os.path.join(ROOT, "profiles", "r02_l2_probe2.txt")
    best = 0.0
    try:
        for ln in open(path):
            f = ln.split()
            if len(f) == 4 and not ln.startswith("#"):
                best = max(best, float(f[3]))
    except OSError:
        return None
    return best * 1e9 or None


def measured_peak():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        return float(json.load(open(p))["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic():
    """Per-launch DRAM bytes per kernel from the committed ncu --set full summary."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(p):
        return json.load(open(p))
    return {}


# ----------------------------------------------------------------- oracle legs
def host_facts():
    """nproc + the CPU model (lscpu), for the oracle's timing context."""
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                model = ln.split(":", 1)[1].strip()
    except (OSError, subprocess.SubprocessError):
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


def pin_one_core():
    """the oracle is timed single-threaded, pinned to one core."""
    try:
        cpu = sorted(os.sched_getaffinity(0))[0]
        prev = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {cpu})
        return cpu, prev
    except (AttributeError, OSError):
        return None, None


def oracle_sample(scale: int, n_src: int = 1, reps_bfs: int = 2):
    """The CPU oracle, as it stands, on an RMAT sample of the same family
    (same generator, seeds and source rule), timed pinned to one core.
    Returns (traversed_edges, seconds, description)."""
    import inputs
    import oracle

    src, dst, w = inputs.rmat_edges(scale, weights=True)
    G = oracle.Graph(1 << scale, src, dst, w)
    deg = G.out_degree()
    srcs = inputs.rmat_sources(scale, max(n_src, reps_bfs))
    total_e, total_s = 0, 0.0
    cpu, prev = pin_one_core()
    for s in srcs[:reps_bfs]:
        t0 = time.perf_counter()
        lv = G.bfs(int(s))
        total_s += time.perf_counter() - t0
        total_e += int(deg[lv != 0xFFFFFFFF].sum())
    for s in srcs[:n_src]:
        t0 = time.perf_counter()
        d = G.sssp(int(s))
        total_s += time.perf_counter() - t0
        total_e += int(deg[d != 0xFFFFFFFF].sum())
    t0 = time.perf_counter()
    G.pagerank(PR_ITERS)
    total_s += time.perf_counter() - t0
    total_e += G.E * PR_ITERS
    for s in srcs[:n_src]:
        lv = G.bfs(int(s))
        t0 = time.perf_counter()
        G.bc([int(s)])
        total_s += time.perf_counter() - t0
        total_e += 2 * int(deg[lv != 0xFFFFFFFF].sum())
    if prev is not None:
        os.sched_setaffinity(0, prev)
    desc = (f"oracle/oracle.c single-threaded, pinned to core {cpu}, on RMAT-{scale} (same "
            f"generator, seeds and source rule, edge factor 16): BFS x{reps_bfs}, SSSP x{n_src}, "
            f"PageRank {PR_ITERS} rounds, BC x{n_src}.  Not the RMAT-28 instance itself: its "
            f"oracle needs ~130 GB of host RAM and ~10 min (tests/test_gpu_fullscale.py "
            f"test_full_oracle), beyond the bench's few-minute bound")
    return total_e, total_s, desc


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import inputs
    import oracle

    scale = 20  # bounded sample per step: a few seconds of single-thread oracle work
    cpu, _ = pin_one_core()
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    G = oracle.Graph(1 << scale, src, dst, w)
    deg = G.out_degree()
    srcs = inputs.rmat_sources(scale, args.warmup + args.steps)

    def step(j):
        s = int(srcs[j])
        e = 0
        lv = G.bfs(s)
        e += int(deg[lv != 0xFFFFFFFF].sum())
        d = G.sssp(s)
        e += int(deg[d != 0xFFFFFFFF].sum())
        G.pagerank(PR_ITERS)
        e += G.E * PR_ITERS
        G.bc([s])
        e += 2 * int(deg[lv != 0xFFFFFFFF].sum())
        return e

    for j in range(args.warmup):
        step(j)
    t0 = time.perf_counter()
    tot = 0
    for j in range(args.steps):
        tot += step(args.warmup + j)
    sec = time.perf_counter() - t0
    val = tot / sec / 1e9
    line = {
        "impl": "reference", "metric": METRIC, "value": val, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * sec / args.steps,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "u32+f64",
        "data": "synthetic",
        # what this arm actually runs: RMAT-20 per step, a bounded sample of our
        # arm's RMAT-28 workload (same generator, seeds, source rule and step)
        "config": {"workload": f"RMAT-{scale} (A,B,C)=(0.57,0.19,0.19) edge factor 16: BFS + "
                               f"SSSP + PageRank x{PR_ITERS} + BC, one source per step",
                   "scale": scale, "vertices": 1 << scale, "edges": 16 << scale,
                   "sample_of": f"RMAT-{args.scale} (our arm's workload; its oracle run is "
                                "minutes per algorithm and ~130 GB of host RAM)",
                   **host_facts()},
        "cpu_baseline": {"value": val, "unit": UNIT, "cores": 1, "kind": "oracle",
                         "sample": f"RMAT-{scale}, one source per step, single thread pinned to "
                                   f"core {cpu}", **host_facts()},
        "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------- our arm
def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    dist = None
    red_dev = "cuda"
    if world > 1:
        import torch.distributed as dist

        # one GPU per rank; TG_DIST_BACKEND=gloo lets several ranks share a GPU
        # (functional testing of the multi-process path on a 1-GPU box)
        backend = os.environ.get("TG_DIST_BACKEND", "nccl")
        torch.cuda.set_device(local % torch.cuda.device_count())
        dist.init_process_group(backend)
        red_dev = "cuda" if backend == "nccl" else "cpu"
    else:
        torch.cuda.set_device(0)
    dev = torch.cuda.current_device()

    import inputs
    import paper_1312_3018_b200 as tg

    scale = args.scale
    V, E = 1 << scale, 16 << scale
    t_build = time.perf_counter()
    comm = tg.TorchComm() if world > 1 else None
    # N > 1: the same graph 1D-partitioned over the N GPUs (one partition per
    # process, boundary messages over NVLink peer copies) -- strong scaling
    eng = tg.Engine.rmat(scale, edge_factor=16, seed=inputs.GRAPH_SEED, wseed=inputs.WEIGHT_SEED,
                         partitions=1, device=dev, weighted=True, in_csr=True, rank=rank,
                         world=world, comm=comm)
    build_s = time.perf_counter() - t_build
    srcs = inputs.rmat_sources(scale, args.warmup + 2 * args.steps + 1)

    lv_d = torch.empty(V, dtype=torch.int32, device="cuda")
    ds_d = torch.empty(V, dtype=torch.int32, device="cuda")
    pr_d = torch.empty(V, dtype=torch.float32, device="cuda")
    bc_d = torch.empty(V, dtype=torch.float64, device="cuda")

    def step(j, outs):
        """One pass of the whole hot path.  Order BC, BFS, PageRank, SSSP: with
        host outputs (e2e) each result's device->host copy overlaps the next
        algorithm, so the largest one (BC, 8 B/vertex) goes first and only the
        last 4 B/vertex copy is left exposed.  Returns stats in bfs, sssp,
        pagerank, bc order."""
        s = int(srcs[j])
        r_bc = eng.bc([s], out=outs[3])[1]
        r_bfs = eng.bfs(s, out=outs[0])[1]
        r_pr = eng.pagerank(PR_ITERS, out=outs[2])[1]
        r_sssp = eng.sssp(s, out=outs[1])[1]
        return [r_bfs, r_sssp, r_pr, r_bc]

    PHASES = ("supersteps", "relaxations", "compute_ms", "exchange_ms", "vote_ms")

    def barrier():
        torch.cuda.synchronize()
        if dist:
            dist.barrier()

    for j in range(args.warmup):
        step(j, (lv_d, ds_d, pr_d, bc_d))

    # ---- device-resident timed region (value) ----
    eng.set_profiling(True)
    per_alg = {"bfs": [0, 0.0], "sssp": [0, 0.0], "pagerank": [0, 0.0], "bc": [0, 0.0]}
    split = {k: {f: 0.0 for f in PHASES} for k in per_alg}
    launches = 0
    barrier()
    with ClockSampler(dev) as clk:
        dev_ms = 0.0
        for j in range(args.steps):
            rs = step(args.warmup + j, (lv_d, ds_d, pr_d, bc_d))
            for name, r in zip(per_alg, rs):
                per_alg[name][0] += r.traversed_edges
                per_alg[name][1] += r.device_ms
                dev_ms += r.device_ms
                launches += r.launches
                for f in PHASES:
                    split[name][f] += getattr(r, f)
        barrier()
    kstats = eng.kernel_stats()
    eng.set_profiling(False)
    # traversed edges are global already (the library all-reduces its stats)
    traversed_all = float(sum(v[0] for v in per_alg.values()))
    ms_step = dev_ms / args.steps
    if dist:  # the slowest rank's device time
        t = torch.tensor([ms_step], device=red_dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_step = float(t.item())
    value = traversed_all / (ms_step * args.steps * 1e-3) / 1e9

    # ---- end to end through the C ABI with host buffers ----
    e2e = None
    if not args.no_e2e:
        def host_set():
            return (torch.empty(V, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                    torch.empty(V, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32),
                    torch.empty(V, dtype=torch.float32, pin_memory=True).numpy(),
                    torch.empty(V, dtype=torch.float64, pin_memory=True).numpy())
        # results copied to the host asynchronously (tg_engine_set_async_collect)
        # into two alternating pinned output sets: each algorithm's copy overlaps
        # the next algorithm, and at the end of step j the collection ticket of
        # step j-1 is waited on -- step j-1's four results are complete in host
        # memory before step j+1 reuses its set; the last step's before the
        # clock stops (tg_engine_sync)
        sets = (host_set(), host_set())
        eng.set_async_collect(world == 1)
        step(args.warmup + 2 * args.steps, sets[1])  # untimed e2e warm-up
        eng.sync()
        barrier()
        t0 = time.perf_counter()
        tr = 0
        prev = eng.last_ticket()
        for j in range(args.steps):
            rs = step(args.warmup + args.steps + j, sets[j % 2])
            eng.wait_ticket(prev)
            prev = eng.last_ticket()
            tr += sum(r.traversed_edges for r in rs)
        eng.sync()
        barrier()
        eng.set_async_collect(False)
        sec = time.perf_counter() - t0
        if dist:
            t = torch.tensor([sec], device=red_dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        e2e = {"value": tr / sec / 1e9, "unit": UNIT,
               # the step's inputs: the source id of BFS, SSSP and BC (8 B each;
               # the graph itself is built once and stays resident in HBM)
               "h2d_bytes_per_step": 3 * 8,
               "d2h_bytes_per_step": V * (4 + 4 + 4 + 8),
               "note": "per step: 3 source ids host->device (BFS, SSSP, BC; the RMAT-28 graph "
                       "is resident in HBM), every per-vertex result (levels, distances, ranks, "
                       "BC scores: 20 B x V) device->pinned host inside the timed region; the "
                       "copies run on the library's copy stream overlapping the next algorithm "
                       "(tg_engine_set_async_collect) into two alternating pinned output sets; "
                       "step j-1's results are waited on (tg_engine_wait_ticket) at the end of "
                       "step j, the last step's (tg_engine_sync) before the clock stops"}

    # ---- roofline of the dominant kernel ----
    peak, peak_src = measured_peak()
    # the dominant HBM kernel (the communication phase is reported separately)
    dom = max((k for k in kstats if k != "exchange_scatter"), key=lambda k: kstats[k]["ms"])
    ks = kstats[dom]
    achieved = ks["algorithmic_bytes"] / (ks["ms"] * 1e-3) / 1e9 if ks["ms"] > 0 else 0.0
    tot_ms = sum(v["ms"] for v in kstats.values())
    traffic = ncu_traffic().get(dom)  # committed ncu --set full capture (per launch)
    roofline = {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                "frac": achieved / peak, "traffic": traffic,
                "traffic_source": "profiles/ncu_traffic.json: dram__bytes_read.sum + "
                                  "dram__bytes_write.sum per launch from a committed ncu "
                                  "capture (pr_pull: the three class pulls averaged over the 5 "
                                  "rounds of one call, profiles/r02_ncu_pr_rounds.csv; not "
                                  "measured inside this run)",
                "algorithmic_bytes_per_launch": ks["algorithmic_bytes"] / max(ks["launches"], 1),
                "avg_launch_ms": ks["ms"] / max(ks["launches"], 1), "peak_source": peak_src,
                "share_of_kernel_time": ks["ms"] / tot_ms if tot_ms else None}
    if dom == "pr_pull":
        # PageRank's pull is bounded by random 4-byte gather requests, not DRAM
        # bytes: the probe (scripts/probes/l2_probe2.cu) measures the B200's rate
        # for its access pattern when every gather hits in L2 -- the ceiling
        ceil = gather_probe_ceiling()
        gps = E / (roofline["avg_launch_ms"] * 1e-3)
        roofline["gather_bound"] = {
            "gathers_per_s": gps, "probe_ceiling_per_s": ceil,
            "frac": gps / ceil if ceil else None,
            "source": "profiles/r02_l2_probe2.txt (index stream + random 4 B gathers, "
                      "L2-resident region, evict_last; ~41 G/s when they miss to HBM)"}
    kernels = {k: {"launches": v["launches"], "ms": round(v["ms"], 3),
                   "GBps": (v["algorithmic_bytes"] / (v["ms"] * 1e-3) / 1e9) if v["ms"] else None}
               for k, v in kstats.items() if v["launches"]}

    # ---- CPU oracle baseline (rank 0, N=1 only) ----
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        e, s, desc = oracle_sample(args.cpu_scale)
        cpu = {"value": e / s / 1e9, "unit": UNIT, "cores": 1, "kind": "oracle", "sample": desc,
               "seconds": s, **host_facts()}

    info = eng.info
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u32+f64", "data": "synthetic",
        "config": {
            "workload": f"RMAT-{scale} (A,B,C)=(0.57,0.19,0.19) edge factor 16: BFS + SSSP + "
                        f"PageRank x{PR_ITERS} + BC, one source per step",
            "scale": scale, "vertices": V, "edges": E, "partitions_per_gpu": 1,
            "parallelism": "single" if world == 1 else
            f"1D vertex partition over {world} GPUs (degree-serpentine); exchange: "
            + ("fused: the compute kernels of all five algorithms write boundary messages into "
               "CUDA-IPC-mapped peer arenas (NVLink stores / reductions)"
               if eng.info["exchange"] == tg.TG_EXCHANGE_FUSED else
               "copy: outbox segments copied into CUDA-IPC-mapped peer arenas")
            + "; vote: shared-memory host collective",
            "l2": "inputs larger than L2 (graph %.1f GB >> 126 MB L2)" % (info["device_bytes"] / 1e9),
            "build_s": round(build_s, 2)},
        "per_algorithm_gteps": {k: (v[0] / (v[1] * 1e-3) / 1e9 if v[1] else None)
                                for k, v in per_alg.items()},
        "per_algorithm_ms_per_step": {k: v[1] / args.steps for k, v in per_alg.items()},
        # supersteps, relaxations and the compute / exchange / vote
        # split per algorithm and step (ledger CUDA events; vote = host time)
        "per_algorithm_phases": {k: {f: v / args.steps for f, v in d.items()}
                                 for k, d in split.items()},
        "e2e": e2e,
        "gpu_launches": launches,
        "roofline": roofline,
        "kernels": kernels,
        "clocks": clk.summary(),
        "cpu_baseline": cpu,
    }
    if rank == 0:
        s = json.dumps(line)
        print(s, flush=True)
        if args.out:
            with open(args.out, "w") as f:
                f.write(s + "\n")
    eng.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
