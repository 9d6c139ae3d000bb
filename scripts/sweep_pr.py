"""PageRank round time on RMAT-s under environment variants of the pull kernels.

usage: sweep_pr.py SCALE VAR=v1;v2;... [VAR2=...]   (cartesian product)
e.g.   sweep_pr.py 28 TG_PR_BATCH=4,4,4;8,8,8 TG_PR_NEXT_HOT=0;16777216
"""
import itertools
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
axes = []
for a in sys.argv[2:]:
    k, v = a.split("=", 1)
    axes.append([(k, x) for x in v.split(";")])
eng = tg.Engine.rmat(scale)
eng.pagerank(2)
for combo in itertools.product(*axes) if axes else [()]:
    for k, v in combo:
        os.environ[k] = v
    ms = [eng.pagerank(5)[1].device_ms / 5 for _ in range(3)]
    tag = " ".join(f"{k}={v}" for k, v in combo)
    print(f"{tag} ms/round={min(ms):.3f} (runs {', '.join(f'{m:.3f}' for m in ms)})", flush=True)
