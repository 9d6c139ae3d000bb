"""SSSP near-far sweep over (Delta, hub degree) at a given scale.

TG_SSSP_DELTA = Delta (0: plain Bellman-Ford); TG_SSSP_HUB_DEG = only rows of
out-degree >= this wait for the near set (0: every row waits).
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, 3)]
os.environ["TG_SSSP_DELTA"] = "0"
refs = [eng.sssp(s)[0].copy() for s in srcs]
grid = [("0", "0")]
for d in sys.argv[2].split(",") if len(sys.argv) > 2 else ("1", "2", "4", "16"):
    for h in sys.argv[3].split(",") if len(sys.argv) > 3 else ("0", "64", "1024"):
        grid.append((d, h))
for d, h in grid:
    os.environ["TG_SSSP_DELTA"] = d
    os.environ["TG_SSSP_HUB_DEG"] = h
    eng.sssp(srcs[0])
    res = [eng.sssp(s) for s in srcs]
    same = all(np.array_equal(r[0], ref) for r, ref in zip(res, refs))
    print(f"delta={d:>3} hub_deg={h:>5} ms={[round(r[1].device_ms, 2) for r in res]} "
          f"steps={[r[1].supersteps for r in res]} "
          f"GB={[r[1].algorithmic_bytes // 10**9 for r in res]} same={same}", flush=True)
