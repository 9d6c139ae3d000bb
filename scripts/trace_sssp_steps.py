import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs, paper_1312_3018_b200 as tg
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
eng = tg.Engine.rmat(scale)
s = int(inputs.rmat_sources(scale, 1)[0])
eng.sssp(s)
eng.set_profiling(True)
os.environ["TG_TRACE"] = "1"
r = eng.sssp(s)[1]
print(r)
print({k: v for k, v in eng.kernel_stats().items() if v["launches"]})
