"""Host facts of the GPU box + oracle timings at a given RMAT scale (to size the
full-oracle RMAT-28 parity test).  Usage: python scripts/box_probe.py [scale]"""
import os
import subprocess
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import inputs  # noqa: E402
import oracle  # noqa: E402

print(subprocess.run("free -g; nproc; lscpu | grep -E 'Model name|Socket|Thread|Core|NUMA node\\(s\\)'; nvidia-smi -L",
                     shell=True, capture_output=True, text=True).stdout)
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 24
V = 1 << scale
t = time.time(); src, dst, w = inputs.rmat_edges(scale, weights=True); print(f"gen {time.time()-t:.1f}s")
t = time.time(); G = oracle.Graph(V, src, dst, w); print(f"csr {time.time()-t:.1f}s")
s = int(inputs.rmat_sources(scale, 1)[0])
for name, f in (("bfs", lambda: G.bfs(s)), ("sssp", lambda: G.sssp(s)), ("pr5", lambda: G.pagerank(5)),
                ("bc1", lambda: G.bc([s]))):
    t = time.time(); f(); print(f"{name} {time.time()-t:.1f}s", flush=True)
