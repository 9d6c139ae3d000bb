"""NEXT-4: boundary-edge ratios (Fig. 4, §3.4) and the
paper's performance model (Eqs. 1-2) recast for P B200s.

For RMAT (0.57, 0.19, 0.19) and UNIFORM (0.25, 0.25, 0.25) at scale s, builds
the engine with P = 2, 3, 4, 8 partitions on one GPU, under the degree-aware
serpentine rule (DEG, reading A23) and the paper's "naive random-based"
baseline (RAND; reading A30), and reads the layout
(tg_engine_partition_info):
  beta_raw = boundary edges / |E|          (no reduction: one message per edge)
  beta_red = outbox slots  / |E|           (source-side reduction)
  balance  = max_p |E_p| / mean_p |E_p|
Model (Eq. 1-2 with c = NVLink message rate, r = one GPU's processing rate),
with a per-superstep latency term lambda that Eq. 1-2 lacks:
  t(G_p) = n_steps * lambda + slots_p / c + |E_p| / r ,  m_P = max_p t(G_p)
  speedup = (|E|/r + n_steps * lambda_1) / m_P
c = 900e9 B/s / msg bytes (4 B per message: level / distance / rank); r and
n_steps (supersteps per run) from a bench JSON of THIS code on one B200 (the
P > 1 path runs the same kernels, direction optimization included, so r is a
rate the P > 1 path achieves); lambda = the multi-process superstep overhead
(arrival barrier + vote through the shared-memory collective + the stream
sync, ~30 us) and lambda_1 = the one-GPU vote (bench phases' vote_ms per
superstep).  Slots and edges are per-run upper bounds (every slot sent, every
edge touched once).
Usage: beta_model.py SCALE [bench.json] [lambda_us]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
bench = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else None
lam = float(sys.argv[3]) * 1e-6 if len(sys.argv) > 3 else 30e-6
C_BYTES = 900e9       # NVLink 5 per direction per GPU (nominal)
MSG = 4               # bytes per boundary message
c = C_BYTES / MSG
print(f"# scale {scale}, E = {16 << scale}; DEG = degree-serpentine (A23), RAND = random (A30)")
print("graph     part  P  beta_raw  beta_red  reduction  edge_balance  max_slots/GPU")
rows = {}
for name, abc in (("RMAT", (0.57, 0.19, 0.19)), ("UNIFORM", (0.25, 0.25, 0.25))):
    for strat, sname in ((tg.TG_PART_DEGREE, "DEG"), (tg.TG_PART_RANDOM, "RAND")):
        for P in (2, 3, 4, 8):
            eng = tg.Engine.rmat(scale, a=abc[0], b=abc[1], c=abc[2], partitions=P, weighted=False,
                                 in_csr=False, strategy=strat)
            E = eng.E
            infos = [eng.partition_info(p) for p in range(P)]
            braw = sum(i["Ep"] - i["Ep_local"] for i in infos) / E
            bred = sum(i["outbox_slots"] for i in infos) / E
            eps = [i["Ep"] for i in infos]
            bal = max(eps) / (sum(eps) / P)
            ms = max(i["outbox_slots"] + i["inbox_slots"] for i in infos)
            rows[(name, sname, P)] = (infos, E)
            print(f"{name:8s} {sname:5s} {P:2d}  {braw:8.4f}  {bred:8.4f}  "
                  f"{braw / max(bred, 1e-12):8.1f}x  {bal:12.4f}  {ms:13d}", flush=True)
            eng.close()
if bench:
    steps = {k: v["supersteps"] for k, v in bench.get("per_algorithm_phases", {}).items()}
    votes = {k: (v["vote_ms"] * 1e-3 / max(v["supersteps"], 1))
             for k, v in bench.get("per_algorithm_phases", {}).items()}
    print(f"\n# model, c = {C_BYTES / 1e9:.0f} GB/s / {MSG} B = {c / 1e9:.0f} G msg/s; lambda = "
          f"{lam * 1e6:.0f} us per superstep at P > 1; r, supersteps and the one-GPU vote from "
          f"{os.path.basename(sys.argv[2])} (scale {bench['config']['scale']})")
    for sname in ("DEG", "RAND"):
        print(f"alg        r(G e/s)  steps   P=2     P=3     P=4     P=8   (predicted speedup, RMAT, "
              f"{sname})")
        for alg, r in bench["per_algorithm_gteps"].items():
            r *= 1e9
            n = steps.get(alg, 10)
            lam1 = votes.get(alg, 0.0)
            # edges touched and slots sent per run: PageRank every round; BC forward + backward
            k = {"pagerank": n, "bc": 2}.get(alg, 1)
            sp = []
            for P in (2, 3, 4, 8):
                infos, E = rows[("RMAT", sname, P)]
                m = max(n * lam + k * (i["outbox_slots"] / c + i["Ep"] / r) for i in infos)
                sp.append((k * E / r + n * lam1) / m)
            print(f"{alg:9s} {r / 1e9:9.1f}  {n:5.1f}  " + "  ".join(f"{x:6.2f}" for x in sp))
