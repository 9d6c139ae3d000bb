"""Full-size parity in the bench launch configuration (RMAT-28, one partition,
device-side generation, the bench's first source).  The oracle cannot hold a
2^32-edge CSR in one thread's time budget, so every output is checked through
properties that hold at any size, evaluated by oracle code over the edge stream
regenerated on the host by the shared input generator:

* BFS levels / SSSP distances: exact O(E) certificates (oracle_*_cert_edges):
  they hold iff the arrays equal the true hop / weighted distances;
* PageRank: the oracle recomputes round 5 from the GPU's round-4 ranks for a
  vertex sample (hubs + random), plus the global mass identity;
* BC (one source): sum_v delta_s(v) = sum_{t reached} (d(s,t) - 1), delta >= 0,
  zero at the source and at unreached vertices.
* CC: every edge joins equal labels, label[v] <= v, label[label[v]] ==
  label[v] (local conditions: they prove labels are constant on components and
  name a member vertex, not that two components were never merged -- exact
  union-find parity is at RMAT-22 in test_gpu_cc.py).

TG_FULL_SCALE=<s> runs the same checks at a smaller scale.
"""
import os
import time

import numpy as np
import pytest

import inputs
import oracle

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
INF = 0xFFFFFFFF


@pytest.fixture(scope="module")
def full():
    import paper_1312_3018_b200 as tg

    scale = int(os.environ.get("TG_FULL_SCALE", "28"))
    V, E = 1 << scale, 16 << scale
    eng = tg.Engine.rmat(scale)                       # bench.py's engine
    s = int(inputs.rmat_sources(scale, 1)[0])          # bench.py's first source
    lv, st_bfs = eng.bfs(s)
    dist, _ = eng.sssp(s)
    r4, _ = eng.pagerank(4)
    r5, _ = eng.pagerank(5)
    bc, _ = eng.bc([s])
    cc, st_cc = eng.cc()
    eng.close()

    t0 = time.time()
    bfs_c = oracle.StreamingCertificate(V, s, lv, weighted=False)
    sssp_c = oracle.StreamingCertificate(V, s, dist, weighted=True)
    outdeg = np.zeros(V, np.uint32)
    indeg = np.zeros(V, np.uint32)
    chunk = 1 << 27
    cc_edges_ok = True
    for first in range(0, E, chunk):                   # pass 1: certificates + degrees
        src, dst, w = inputs.rmat_edges(scale, weights=True, first=first,
                                        count=min(chunk, E - first))
        bfs_c.feed(src, dst)
        sssp_c.feed(src, dst, w)
        oracle.outdeg_edges(V, src, outdeg)
        oracle.outdeg_edges(V, dst, indeg)
        cc_edges_ok = cc_edges_ok and bool(np.array_equal(cc[src], cc[dst]))
    rng = np.random.default_rng(2024)
    sample = np.unique(np.concatenate([np.argsort(indeg)[-256:], rng.integers(0, V, 8192)]))
    mask = np.zeros((V + 63) // 64, np.uint64)
    np.bitwise_or.at(mask, sample >> 6, np.uint64(1) << (sample & 63).astype(np.uint64))
    slot = np.zeros(V, np.uint32)
    slot[sample] = np.arange(len(sample), dtype=np.uint32)
    acc = np.zeros(len(sample))
    for first in range(0, E, chunk):                   # pass 2: PageRank sample recurrence
        src, dst, _ = inputs.rmat_edges(scale, first=first, count=min(chunk, E - first))
        oracle.pr_sample_edges(V, src, dst, mask, slot, r4, outdeg, acc)
    print(f"full-scale host checks: {time.time() - t0:.1f} s")
    return dict(scale=scale, V=V, E=E, s=s, lv=lv, dist=dist, r4=r4, r5=r5, bc=bc, bfs_c=bfs_c,
                sssp_c=sssp_c, outdeg=outdeg, indeg=indeg, sample=sample, acc=acc, st_bfs=st_bfs,
                cc=cc, st_cc=st_cc, cc_edges_ok=cc_edges_ok)


def test_full_bfs_certificate(full):
    assert full["lv"][full["s"]] == 0
    assert full["bfs_c"].holds()
    reached = full["lv"] != INF
    assert full["st_bfs"].traversed_edges == int(full["outdeg"][reached].sum())


def test_full_sssp_certificate(full):
    assert full["sssp_c"].holds()
    # every vertex BFS reaches SSSP reaches, and vice versa
    assert np.array_equal(full["lv"] != INF, full["dist"] != INF)


def test_full_pagerank_recurrence_and_mass(full):
    d, V = 0.85, full["V"]
    pred = (1 - d) / V + d * full["acc"]
    got = full["r5"][full["sample"]].astype(np.float64)
    rel = np.abs(got - pred) / pred
    assert rel.max() <= 1e-5, rel.max()
    nondangling = full["outdeg"] > 0
    mass_pred = (1 - d) + d * full["r4"][nondangling].astype(np.float64).sum()
    assert abs(full["r5"].astype(np.float64).sum() - mass_pred) <= 1e-5 * mass_pred


def test_full_bc_dependency_identity(full):
    lv, bc, s = full["lv"].astype(np.int64), full["bc"], full["s"]
    reached = (full["lv"] != INF) & (np.arange(full["V"]) != s)
    expect = float((lv[reached] - 1).sum())
    assert abs(bc.sum() - expect) <= 1e-6 * max(expect, 1.0)
    assert (bc >= 0).all() and bc[s] == 0
    assert (bc[full["lv"] == INF] == 0).all()


def test_full_cc_local_certificate(full):
    cc, V = full["cc"], full["V"]
    assert full["cc_edges_ok"]
    assert (cc <= np.arange(V, dtype=np.uint32)).all()
    assert np.array_equal(cc[cc], cc)
    isolated = (full["outdeg"] == 0) & (full["indeg"] == 0)
    assert np.array_equal(cc[isolated], np.flatnonzero(isolated).astype(np.uint32))
    assert full["st_cc"].traversed_edges == full["E"]


@pytest.mark.skipif(os.environ.get("TG_RMAT30") != "1",
                    reason="RMAT-30 (2^34 edges, ~15 min of host certificate work): TG_RMAT30=1")
def test_rmat30_bfs_certificate_one_gpu():
    """BASELINE configs[4]'s graph (RMAT-30, 17.2 G edges) on ONE B200: an
    out-CSR-only engine (no weights, no in-CSR: ~100 GB) runs top-down BFS from
    the bench's first source; the exact streaming certificate over the
    regenerated 2^34-edge stream proves every level."""
    import paper_1312_3018_b200 as tg

    scale = 30
    V, E = 1 << scale, 16 << scale
    eng = tg.Engine.rmat(scale, weighted=False, in_csr=False)
    s = int(inputs.rmat_sources(scale, 1)[0])
    lv, st = eng.bfs(s)
    eng.close()
    cert = oracle.StreamingCertificate(V, s, lv, weighted=False)
    chunk = 1 << 28
    for first in range(0, E, chunk):
        src, dst, _ = inputs.rmat_edges(scale, first=first, count=min(chunk, E - first))
        cert.feed(src, dst)
    assert cert.holds()
    print(f"RMAT-30 BFS: {st.device_ms:.1f} ms, supersteps {st.supersteps}, "
          f"{st.traversed_edges / st.device_ms / 1e6:.1f} GTEPS")
