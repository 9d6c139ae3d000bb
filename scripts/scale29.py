"""Capacity check beyond C4: RMAT-29 (2^29 vertices, 2^33 edges) on ONE B200,
unweighted, with the in-CSR: BFS from the first bench source and PageRank x5."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 29
t = time.time()
eng = tg.Engine.rmat(scale, weighted=False)
print(f"RMAT-{scale}: V={eng.V} E={eng.E} build {time.time() - t:.1f} s, device {eng.info['device_bytes'] / 1e9:.1f} GB",
      flush=True)
s = int(inputs.rmat_sources(scale, 1)[0])
for _ in range(2):
    lv, st = eng.bfs(s)
    print(f"bfs {st.device_ms:.2f} ms, {st.traversed_edges / st.device_ms / 1e6:.1f} GTEPS, supersteps {st.supersteps}",
          flush=True)
for _ in range(2):
    r, st = eng.pagerank(5)
    print(f"pagerank x5 {st.device_ms:.2f} ms, {st.traversed_edges / st.device_ms / 1e6:.1f} G edges/s",
          flush=True)
import numpy as np  # noqa: E402
print(f"sum of ranks {float(np.sum(r, dtype=np.float64)):.6f}, reached {(lv != 0xFFFFFFFF).sum()}", flush=True)
