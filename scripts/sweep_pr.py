"""PageRank round time vs the evict_last hub prefix (TG_PR_HOT)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
eng = tg.Engine.rmat(scale)
eng.pagerank(2)
for hot in ("0", str(1 << 20), str(4 << 20), str(8 << 20), str(16 << 20), str(24 << 20), str(1 << 31)):
    os.environ["TG_PR_HOT"] = hot
    ms = [eng.pagerank(5)[1].device_ms / 5 for _ in range(2)]
    print(f"hot={hot} ms/round={min(ms):.2f}", flush=True)
