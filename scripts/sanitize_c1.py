"""Small run of all five algorithms for compute-sanitizer (memcheck /
racecheck / synccheck): SPEC C1 (RMAT-10) at P = 1, 2 and 3 (per-partition streams) in both exchange
transports, direction modes auto; each result is checked against the oracle so
a sanitizer run is also a parity run.

usage: compute-sanitizer --tool memcheck python scripts/sanitize_c1.py
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import oracle  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(os.environ.get("TG_SAN_SCALE", "10"))
src, dst, w = inputs.rmat_edges(scale, weights=True)
V = 1 << scale
G = oracle.Graph(V, src, dst, w)
s = int(inputs.rmat_sources(scale, 1)[0])
ref = {"bfs": G.bfs(s), "sssp": G.sssp(s), "pr": G.pagerank(5), "bc": G.bc([s]), "cc": G.cc()}
for P in (1, 2, 3):
    for x in ((None,) if P == 1 else (tg.TG_EXCHANGE_FUSED, tg.TG_EXCHANGE_COPY)):
        eng = tg.Engine.rmat(scale, partitions=P)
        if x is not None:
            eng.set_exchange(x)
        assert np.array_equal(eng.bfs(s)[0], ref["bfs"])
        assert np.array_equal(eng.sssp(s)[0], ref["sssp"])
        assert (np.abs(eng.pagerank(5)[0] - ref["pr"]) / ref["pr"]).max() <= 1e-5
        b = eng.bc([s])[0]
        assert np.allclose(b, ref["bc"], rtol=1e-4, atol=1e-12 * max(1.0, ref["bc"].max()))
        assert np.array_equal(eng.cc()[0], ref["cc"])
        if P == 2:
            eng.set_pagerank_comm(tg.TG_PR_PULL)
            assert (np.abs(eng.pagerank(5)[0] - ref["pr"]) / ref["pr"]).max() <= 1e-5
        eng.close()
        print(f"P={P} exchange={x}: ok", flush=True)
print("sanitize_c1 done")
