"""Device time per algorithm (BFS, SSSP, BC from one source; PageRank 5 rounds)
on RMAT-s, best of 3 after a warm-up; one line, tagged with argv[2]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
tag = sys.argv[2] if len(sys.argv) > 2 else ""
eng = tg.Engine.rmat(scale)
s = int(inputs.rmat_sources(scale, 1)[0])
run = {"bfs": lambda: eng.bfs(s), "sssp": lambda: eng.sssp(s), "bc": lambda: eng.bc([s]),
       "pr5": lambda: eng.pagerank(5)}
out = {}
for a, f in run.items():
    f()
    out[a] = min(f()[1].device_ms for _ in range(3))
print(tag, " ".join(f"{a}={v:.3f}ms" for a, v in out.items()), flush=True)
