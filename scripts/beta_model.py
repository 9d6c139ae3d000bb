"""NEXT-4: boundary-edge ratios (Fig. 4, §3.4) and the
paper's performance model (Eqs. 1-2) recast for P B200s.

For RMAT (0.57, 0.19, 0.19) and UNIFORM (0.25, 0.25, 0.25) at scale s, builds
the engine with P = 2, 3, 4, 8 degree-serpentine partitions on one GPU and
reads the layout (tg_engine_partition_info):
  beta_raw = boundary edges / |E|          (no reduction: one message per edge)
  beta_red = outbox slots  / |E|           (source-side reduction)
  balance  = max_p |E_p| / mean_p |E_p|
Model (Eq. 1-2 with c = NVLink message rate, r = one GPU's processing rate):
  t(G_p) = slots_p / c + |E_p| / r ,  m_P = max_p t(G_p),  speedup = (|E|/r) / m_P
with c = 900e9 B/s / msg bytes (4 B per message: level / distance / rank), r from
a bench JSON (per_algorithm_gteps, edges/s of one B200), per superstep summed
over the supersteps the algorithm runs (slots and edges are per superstep
upper bounds: every slot sent, every edge touched once per run).
Usage: beta_model.py SCALE [bench.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
bench = json.load(open(sys.argv[2])) if len(sys.argv) > 2 else None
C_BYTES = 900e9       # NVLink 5 per direction per GPU (nominal)
MSG = 4               # bytes per boundary message
c = C_BYTES / MSG
print(f"# scale {scale}, E = {16 << scale}, degree-serpentine partitions (A23)")
print("graph     P  beta_raw  beta_red  reduction  edge_balance  max_slots/GPU")
rows = {}
for name, abc in (("RMAT", (0.57, 0.19, 0.19)), ("UNIFORM", (0.25, 0.25, 0.25))):
    for P in (2, 3, 4, 8):
        eng = tg.Engine.rmat(scale, a=abc[0], b=abc[1], c=abc[2], partitions=P, weighted=False,
                             in_csr=False)
        E = eng.E
        infos = [eng.partition_info(p) for p in range(P)]
        braw = sum(i["Ep"] - i["Ep_local"] for i in infos) / E
        bred = sum(i["outbox_slots"] for i in infos) / E
        eps = [i["Ep"] for i in infos]
        bal = max(eps) / (sum(eps) / P)
        ms = max(i["outbox_slots"] + i["inbox_slots"] for i in infos)
        rows[(name, P)] = (infos, E)
        print(f"{name:8s} {P:2d}  {braw:8.4f}  {bred:8.4f}  {braw / max(bred, 1e-12):8.1f}x  "
              f"{bal:12.4f}  {ms:13d}")
        eng.close()
if bench:
    print(f"\n# model, c = {C_BYTES / 1e9:.0f} GB/s / {MSG} B = {c / 1e9:.0f} G msg/s; r = one B200's "
          f"rate from {os.path.basename(sys.argv[2])} (scale {bench['config']['scale']})")
    print("alg        r(G e/s)   P=2     P=3     P=4     P=8   (predicted speedup over 1 GPU, RMAT)")
    for alg, r in bench["per_algorithm_gteps"].items():
        r *= 1e9
        sp = []
        for P in (2, 3, 4, 8):
            infos, E = rows[("RMAT", P)]
            m = max(i["outbox_slots"] / c + i["Ep"] / r for i in infos)
            sp.append((E / r) / m)
        print(f"{alg:9s} {r / 1e9:9.1f}  " + "  ".join(f"{x:6.2f}" for x in sp))
