"""Device ms per algorithm with P partitions hosted on one GPU, COPY vs FUSED
exchange (tg_engine_set_exchange), RMAT-s; best of 3 after a warm-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
P = int(sys.argv[2]) if len(sys.argv) > 2 else 4
eng = tg.Engine.rmat(scale, partitions=P)
s = int(inputs.rmat_sources(scale, 1)[0])
run = {"bfs": lambda: eng.bfs(s), "sssp": lambda: eng.sssp(s), "pr5": lambda: eng.pagerank(5),
       "bc": lambda: eng.bc([s]), "cc": lambda: eng.cc()}
for mode, name in ((tg.TG_EXCHANGE_COPY, "COPY"), (tg.TG_EXCHANGE_FUSED, "FUSED")):
    eng.set_exchange(mode)
    out = {}
    for a, f in run.items():
        f()
        out[a] = min(f()[1].device_ms for _ in range(3))
    print(f"scale {scale} P={P} {name}: " + " ".join(f"{a}={v:.3f}ms" for a, v in out.items()), flush=True)
