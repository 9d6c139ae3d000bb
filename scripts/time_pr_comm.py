"""PageRank x5 device ms with P partitions on one GPU: push partial sums vs
ghost-pull (tg_engine_set_pagerank_comm), RMAT-s; communicated bytes per run."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
for P in [int(x) for x in (sys.argv[2] if len(sys.argv) > 2 else "2,4,8").split(",")]:
    eng = tg.Engine.rmat(scale, partitions=P, weighted=False)
    for mode, name in ((tg.TG_PR_PUSH, "push"), (tg.TG_PR_PULL, "pull")):
        eng.set_pagerank_comm(mode)
        eng.pagerank(5)
        runs = [eng.pagerank(5)[1] for _ in range(3)]
        best = min(runs, key=lambda r: r.device_ms)
        print(f"scale {scale} P={P} {name}: pr5={best.device_ms:.3f} ms comm_bytes={best.comm_bytes}",
              flush=True)
    eng.close()
