"""Per-superstep trace (TG_TRACE=1: counts + synchronized lap ms) of BFS, SSSP
and BC from one source, plus the kernel ledger of each, at a given scale.
usage: trace_all.py SCALE [algs] [P]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
algs = sys.argv[2].split(",") if len(sys.argv) > 2 else ["bfs", "sssp", "bc"]
P = int(sys.argv[3]) if len(sys.argv) > 3 else 1
eng = tg.Engine.rmat(scale, partitions=P)
s = int(inputs.rmat_sources(scale, 1)[0])
run = {"bfs": lambda: eng.bfs(s), "sssp": lambda: eng.sssp(s), "bc": lambda: eng.bc([s]),
       "pagerank": lambda: eng.pagerank(5)}
for a in algs:
    run[a]()  # warm
    eng.set_profiling(True)
    r = run[a]()[1]
    eng.set_profiling(False)
    print(f"== {a} untraced: {r.device_ms:.3f} ms", flush=True)
    print({k: round(v["ms"], 3) for k, v in eng.kernel_stats().items() if v["launches"]}, flush=True)
    os.environ["TG_TRACE"] = "1"
    run[a]()
    os.environ["TG_TRACE"] = "0"
    sys.stderr.flush()
