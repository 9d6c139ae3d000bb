"""CC device ms on RMAT-s (best of 3 after a warm-up), tagged with argv[2]."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 28
eng = tg.Engine.rmat(scale)
eng.cc()
r = [eng.cc()[1] for _ in range(3)]
print(sys.argv[2] if len(sys.argv) > 2 else "", f"cc={min(x.device_ms for x in r):.3f}ms supersteps={r[0].supersteps}",
      flush=True)
