"""Host-output collection cost: BFS / PageRank / BC wall ms with pinned host
outputs minus the device-output call, per TG_COLLECT mode (RMAT-s)."""
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
hu = torch.empty(V, dtype=torch.int32, pin_memory=True).numpy().view("uint32")
hf = torch.empty(V, dtype=torch.float32, pin_memory=True).numpy()
hd = torch.empty(V, dtype=torch.float64, pin_memory=True).numpy()
du = torch.empty(V, dtype=torch.int32, device="cuda")
dd = torch.empty(V, dtype=torch.float64, device="cuda")


def wall(f):
    f()
    torch.cuda.synchronize()
    best = 1e9
    for _ in range(3):
        t = time.perf_counter()
        f()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best * 1e3


for mode in ("0", "1", "2"):
    os.environ["TG_COLLECT"] = mode
    b_h, b_d = wall(lambda: eng.bfs(s, out=hu)), wall(lambda: eng.bfs(s, out=du))
    c_h, c_d = wall(lambda: eng.bc([s], out=hd)), wall(lambda: eng.bc([s], out=dd))
    print(f"TG_COLLECT={mode}: bfs host {b_h:.1f} dev {b_d:.1f} (collect u32 to host ~{b_h - b_d:.1f} ms, "
          f"{4 * V / (b_h - b_d) / 1e6:.1f} GB/s); bc host {c_h:.1f} dev {c_d:.1f} (f64 ~{c_h - c_d:.1f} ms, "
          f"{8 * V / (c_h - c_d) / 1e6:.1f} GB/s)", flush=True)
