"""Small driver for ncu captures: one BFS, SSSP, PageRank round and BC on RMAT-s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
algs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bfs", "sssp", "pr", "bc"]
eng = tg.Engine.rmat(scale)
s = int(inputs.rmat_sources(scale, 1)[0])
for a in algs:
    if a == "bfs":
        print("bfs", eng.bfs(s)[1])
    elif a == "sssp":
        print("sssp", eng.sssp(s)[1])
    elif a == "pr":
        print("pr", eng.pagerank(1)[1])
    elif a == "bc":
        print("bc", eng.bc([s])[1])
