"""A/B of BUILD-time environment switches (read when the engine is built):
scripts/ab_build_env.py SCALE VAR=a;b -- a fresh engine per value; device ms of
BFS / SSSP / BC (bench's first source) and PageRank x5, best of 3 after a warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1])
k, vals = sys.argv[2].split("=", 1)
s = int(inputs.rmat_sources(scale, 1)[0])
for v in vals.split(";"):
    os.environ[k] = v
    eng = tg.Engine.rmat(scale)
    run = {"bfs": lambda: eng.bfs(s), "sssp": lambda: eng.sssp(s), "bc": lambda: eng.bc([s]),
           "pr5": lambda: eng.pagerank(5)}
    out = {}
    for a, f in run.items():
        f()
        out[a] = min(f()[1].device_ms for _ in range(3))
    print(f"{k}={v}", " ".join(f"{a}={x:.3f}ms" for a, x in out.items()), flush=True)
    eng.close()
