"""Wall ms per C-ABI call with pinned host outputs in the bench's step order
(BC, BFS, PageRank, SSSP), synchronous vs asynchronous collection
(tg_engine_set_async_collect), plus the final tg_engine_sync wait."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
V = 1 << scale
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, 14)]
lv = torch.empty(V, dtype=torch.int32, pin_memory=True).numpy().view("uint32")
ds = torch.empty(V, dtype=torch.int32, pin_memory=True).numpy().view("uint32")
pr = torch.empty(V, dtype=torch.float32, pin_memory=True).numpy()
bc = torch.empty(V, dtype=torch.float64, pin_memory=True).numpy()
for on in (False, True, False, True):
    eng.set_async_collect(on)
    for j in (8, 9, 10):
        s = srcs[j]
        t = [time.perf_counter()]
        r = [eng.bc([s], out=bc)[1]]; t.append(time.perf_counter())
        r.append(eng.bfs(s, out=lv)[1]); t.append(time.perf_counter())
        r.append(eng.pagerank(5, out=pr)[1]); t.append(time.perf_counter())
        r.append(eng.sssp(s, out=ds)[1]); t.append(time.perf_counter())
        eng.sync(); t.append(time.perf_counter())
        w = [(t[i + 1] - t[i]) * 1e3 for i in range(5)]
        print(f"async={int(on)} j={j} wall ms bc/bfs/pr/sssp/sync = " + "/".join(f"{x:.1f}" for x in w) +
              "  device ms = " + "/".join(f"{x.device_ms:.1f}" for x in r) + f"  total {sum(w):.1f}",
              flush=True)
