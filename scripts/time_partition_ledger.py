"""P partitions on one GPU: device ms per algorithm vs the summed kernel time of
its ledger (tg_engine_set_profiling), to separate kernel work from the gaps
between the per-partition launches.  usage: time_partition_ledger.py SCALE P..."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import inputs  # noqa: E402
import paper_1312_3018_b200 as tg  # noqa: E402

scale = int(sys.argv[1])
for P in [int(x) for x in sys.argv[2:]]:
    eng = tg.Engine.rmat(scale, partitions=P)
    s = int(inputs.rmat_sources(scale, 1)[0])
    for name, f in (("bfs", lambda: eng.bfs(s)), ("sssp", lambda: eng.sssp(s)),
                    ("pagerank", lambda: eng.pagerank(5)), ("bc", lambda: eng.bc([s]))):
        f()
        plain = min(f()[1].device_ms for _ in range(3))
        eng.set_profiling(True)
        st = f()[1]
        ks = eng.kernel_stats()
        eng.set_profiling(False)
        kern = sum(v["ms"] for v in ks.values())
        print(f"scale {scale} P={P} {name}: device {plain:.3f} ms, ledger kernel sum {kern:.3f} ms "
              f"(compute {st.compute_ms:.3f}, exchange {st.exchange_ms:.3f}), supersteps "
              f"{st.supersteps}, launches {st.launches}", flush=True)
    eng.close()
