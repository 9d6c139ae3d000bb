"""SSSP device ms on RMAT-s vs the near-far schedule (TG_SSSP_DELTA x
TG_SSSP_HUB_DEG), mean over the bench's first 3 sources (best of 2 each)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
deltas = (sys.argv[2] if len(sys.argv) > 2 else "0,1,2,4").split(",")
hubs = (sys.argv[3] if len(sys.argv) > 3 else "32,128,512").split(",")
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, 3)]
eng.sssp(srcs[0])
for d in deltas:
    for h in hubs:
        os.environ["TG_SSSP_DELTA"], os.environ["TG_SSSP_HUB_DEG"] = d, h
        ms = [min(eng.sssp(s)[1].device_ms for _ in range(2)) for s in srcs]
        print(f"delta={d} hub_deg={h} mean_ms={sum(ms) / len(ms):.3f} ({', '.join(f'{m:.2f}' for m in ms)})",
              flush=True)
        if d == "0":
            break
