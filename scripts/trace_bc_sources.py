"""BC device ms per source (bench sources j = 0..n-1) on RMAT-s, with the
per-level trace (TG_TRACE=1) on stderr for the second run of each."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
n = int(sys.argv[2]) if len(sys.argv) > 2 else 6
eng = tg.Engine.rmat(scale)
srcs = [int(x) for x in inputs.rmat_sources(scale, n)]
eng.bc([srcs[0]])
for j, s in enumerate(srcs):
    a = eng.bc([s])[1]
    os.environ["TG_TRACE"] = "1"
    print(f"--- j={j} source={s}", file=sys.stderr, flush=True)
    eng.bc([s])
    os.environ["TG_TRACE"] = "0"
    print(f"j={j} source={s} bc_ms={a.device_ms:.3f} supersteps={a.supersteps} teps_edges={a.traversed_edges}",
          flush=True)
