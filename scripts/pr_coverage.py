"""Share of a PageRank round's gathers that the top-K sources (in out-degree
order, the engine's local-id order) serve, on the RMAT graph of the given
scale: sizes the hub prefix a shared-memory replica can hold.  Also the
in-degree class split (thread < 32 <= warp < 2048 <= CTA) of rows and edges.
usage: pr_coverage.py SCALE"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
V, E = 1 << scale, 16 << scale
dev = torch.device("cuda", 0)
outd = torch.zeros(V, dtype=torch.int32, device=dev)
ind = torch.zeros(V, dtype=torch.int32, device=dev)
chunk = 1 << 28
src = torch.empty(chunk, dtype=torch.int32, device=dev)
dst = torch.empty(chunk, dtype=torch.int32, device=dev)
one = torch.ones(chunk, dtype=torch.int32, device=dev)
for first in range(0, E, chunk):
    n = min(chunk, E - first)
    tg.tg_rmat_edges(scale, first=first, count=n, out=(src[:n], dst[:n], None))
    outd.index_add_(0, src[:n].long(), one[:n])
    ind.index_add_(0, dst[:n].long(), one[:n])
od = torch.sort(outd, descending=True).values.to(torch.int64)
cum = torch.cumsum(od, 0)
print(f"RMAT-{scale}: V={V} E={E}")
for K in (1024, 4096, 8192, 16384, 24576, 32768, 49152, 53248, 57344, 65536, 131072, 262144,
          1 << 20, 4 << 20, 8 << 20, 16 << 20, 32 << 20):
    if K <= V:
        print(f"top {K:>10d} sources ({K * 4 / 2**20:8.2f} MB fp32): {cum[K - 1].item() / E:.4f} of edges")
ind64 = ind.to(torch.int64)
for lo, hi, name in ((0, 32, "thread"), (32, 2048, "warp"), (2048, 1 << 40, "cta")):
    m = (ind64 >= lo) & (ind64 < hi)
    print(f"class {name}: rows {m.sum().item()}, edges {ind64[m].sum().item() / E:.4f}")
