"""Device-side permutation cost of the result collection (degree order ->
global order): wall ms of a device-output call minus its device_ms, per
TG_COLLECT mode (1 gather, 3 binned two-pass), RMAT-s; best of 3."""
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
s = int(inputs.rmat_sources(scale, 1)[0])
du = torch.empty(V, dtype=torch.int32, device="cuda")
dd = torch.empty(V, dtype=torch.float64, device="cuda")


def extra(f):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        st = f()[1]
        torch.cuda.synchronize()
        best = min(best, (time.perf_counter() - t) * 1e3 - st.device_ms)
    return best


for mode in sys.argv[2:] if len(sys.argv) > 2 else ("1", "3", "1", "3"):
    os.environ["TG_COLLECT"] = mode
    b = extra(lambda: eng.bfs(s, out=du))
    c = extra(lambda: eng.bc([s], out=dd))
    print(f"TG_COLLECT={mode}: outside device_ms: bfs (u32) {b:.2f} ms, bc (f64) {c:.2f} ms", flush=True)
