"""Direction-optimization thresholds: BFS (TG_BU_ALPHA x TG_BU_BETA) and BC
(TG_BC_ALPHA), mean device ms over the bench's first 6 sources (RMAT-s)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, 6)]
eng.bfs(srcs[0]); eng.bc([srcs[0]])


def mean(f):
    return sum(min(f(s)[1].device_ms for _ in range(2)) for s in srcs) / len(srcs)


for a in ("6", "14", "24"):
    for b in ("12", "24", "64"):
        os.environ["TG_BU_ALPHA"], os.environ["TG_BU_BETA"] = a, b
        print(f"bfs alpha={a} beta={b} mean_ms={mean(lambda s: eng.bfs(s)):.3f}", flush=True)
os.environ["TG_BU_ALPHA"], os.environ["TG_BU_BETA"] = "14", "24"
for a in ("1", "2", "4", "8"):
    os.environ["TG_BC_ALPHA"] = a
    print(f"bc alpha={a} mean_ms={mean(lambda s: eng.bc([s])):.3f}", flush=True)
