"""Device ms of BFS / SSSP / BC per bench source j (RMAT-s)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = int(sys.argv[2]) if len(sys.argv) > 2 else 14
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, n)]
eng.bfs(srcs[0]); eng.sssp(srcs[0]); eng.bc([srcs[0]])
for j, s in enumerate(srcs):
    b, ss, c = eng.bfs(s)[1], eng.sssp(s)[1], eng.bc([s])[1]
    print(f"j={j} bfs={b.device_ms:.2f} (L={b.supersteps}) sssp={ss.device_ms:.2f} (steps={ss.supersteps}) "
          f"bc={c.device_ms:.2f} (steps={c.supersteps}) reached_edges={b.traversed_edges}", flush=True)
