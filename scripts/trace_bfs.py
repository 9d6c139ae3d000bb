"""Per-superstep trace of BFS / BC at a given scale and direction settings."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, 3)]
eng.bfs(srcs[0])
os.environ["TG_TRACE"] = "1"
print("auto bfs ms", [round(eng.bfs(s)[1].device_ms, 2) for s in srcs], flush=True)
print("auto bc ms", [round(eng.bc([s])[1].device_ms, 2) for s in srcs], flush=True)
os.environ["TG_TRACE"] = "0"
for a in ("1", "4", "30", "100"):
    os.environ["TG_BU_ALPHA"] = a
    os.environ["TG_BC_ALPHA"] = a
    print("alpha", a, "bfs", [round(eng.bfs(s)[1].device_ms, 2) for s in srcs],
          "bc", [round(eng.bc([s])[1].device_ms, 2) for s in srcs], flush=True)
os.environ["TG_DIRECTION"] = "top"
print("top-down bfs ms", [round(eng.bfs(s)[1].device_ms, 2) for s in srcs])
print("top-down bc ms", [round(eng.bc([s])[1].device_ms, 2) for s in srcs])
