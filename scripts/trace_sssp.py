"""SSSP near-far Delta sweep at a given scale."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, 3)]
ref = eng.sssp(srcs[0])[0].copy()
for d in ("0", "16", "32", "64", "128", "256", "512"):
    os.environ["TG_SSSP_DELTA"] = d
    res = [eng.sssp(s) for s in srcs]
    import numpy as np
    same = np.array_equal(eng.sssp(srcs[0])[0], ref)
    print(f"delta={d} ms={[round(r[1].device_ms, 2) for r in res]} steps={[r[1].supersteps for r in res]} "
          f"relax_bytes={[r[1].algorithmic_bytes // 10**9 for r in res]}GB same={same}", flush=True)
