"""SSSP on RMAT-s: dense-step next-frontier marking (TG_SSSP_DENSE_DIV) A/B, ms per run
over the bench's first sources, interleaved variants (same box, same engine)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
eng = tg.Engine.rmat(scale)
srcs = [int(s) for s in inputs.rmat_sources(scale, 4)]
eng.sssp(srcs[0])
res = {}
for rep in range(2):
    for div in ("0", "64", "16", "256"):
        os.environ["TG_SSSP_DENSE_DIV"] = div
        for s in srcs:
            st = eng.sssp(s)[1]
            res.setdefault(div, []).append(st.device_ms)
for div, ms in res.items():
    print(f"TG_SSSP_DENSE_DIV={div} mean ms={sum(ms) / len(ms):.3f} min={min(ms):.3f} runs={len(ms)}")
