"""Generic A/B of run-time environment switches: scripts/sweep_env.py SCALE
VAR=a;b [VAR2=...] -- device ms of BFS/SSSP/BC (bench's first source) and
PageRank x5 for every combination, best of 3 after a warm-up."""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1])
axes = [[(k, x) for x in v.split(";")] for k, v in (a.split("=", 1) for a in sys.argv[2:])]
eng = tg.Engine.rmat(scale)
s = int(inputs.rmat_sources(scale, 1)[0])
run = {"bfs": lambda: eng.bfs(s), "sssp": lambda: eng.sssp(s), "bc": lambda: eng.bc([s]),
       "pr5": lambda: eng.pagerank(5)}
for combo in itertools.product(*axes):
    for k, v in combo:
        os.environ[k] = v
    out = {}
    for a, f in run.items():
        f()
        out[a] = min(f()[1].device_ms for _ in range(3))
    print(" ".join(f"{k}={v}" for k, v in combo), " ".join(f"{a}={v:.3f}ms" for a, v in out.items()),
          flush=True)
