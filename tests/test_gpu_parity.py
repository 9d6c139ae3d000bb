"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle on the
same seeded inputs.  Bars (BASELINE.json north_star): BFS levels and SSSP
distances bit-exact; PageRank within 1e-5 relative per vertex; BC within 1e-4
relative per vertex."""
import functools
import json
import os

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
PR_RTOL = 1e-5
BC_RTOL = 1e-4


@pytest.fixture(scope="module")
def tg():
    import paper_1312_3018_b200 as tg

    tg.lib()
    return tg


def assert_pr(gpu, ref):
    rel = np.abs(gpu.astype(np.float64) - ref) / np.abs(ref)
    assert rel.max() <= PR_RTOL, f"PageRank max rel err {rel.max():.3e} at {rel.argmax()}"


def assert_bc(gpu, ref):
    scale = max(1.0, float(np.abs(ref).max()))
    err = np.abs(gpu - ref)
    ok = err <= BC_RTOL * np.abs(ref) + 1e-12 * scale
    assert ok.all(), f"BC mismatch at {np.where(~ok)[0][:5]}: {gpu[~ok][:5]} vs {ref[~ok][:5]}"


def both(tg, V, src, dst, w=None, P=1):
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.from_edges(V, np.asarray(src, np.uint32), np.asarray(dst, np.uint32),
                               None if w is None else np.asarray(w, np.uint32), partitions=P,
                               weighted=w is not None)
    return G, eng


def check_all(tg, G, eng, bfs_src=(), sssp_src=(), pr_T=(5,), bc_src=()):
    for s in bfs_src:
        lv, st = eng.bfs(int(s))
        assert np.array_equal(lv, G.bfs(int(s))), f"BFS mismatch from {s}"
    for s in sssp_src:
        d, _ = eng.sssp(int(s))
        assert np.array_equal(d, G.sssp(int(s))), f"SSSP mismatch from {s}"
    for T in pr_T:
        r, _ = eng.pagerank(T)
        assert_pr(r, G.pagerank(T))
    if len(bc_src):
        b, _ = eng.bc(np.asarray(bc_src, np.uint64))
        assert_bc(b, G.bc(bc_src))


# ------------------------------------------------------------ SPEC worked examples
@pytest.mark.parametrize("P", [1, 2])
def test_golden(tg, P):
    g = GOLD["bfs_path_split"]
    G, eng = both(tg, g["V"], g["src"], g["dst"], P=P)
    assert eng.bfs(g["source"])[0].tolist() == g["levels"], g["cite"]
    g = GOLD["bfs_isolated_source"]
    G, eng = both(tg, g["V"], g["src"], g["dst"], P=P)
    assert eng.bfs(g["source"])[0].tolist() == g["levels"], g["cite"]
    g = GOLD["sssp_triangle"]
    G, eng = both(tg, g["V"], g["src"], g["dst"], g["w"], P=P)
    assert eng.sssp(g["source"])[0].tolist() == g["dist"], g["cite"]
    g = GOLD["pagerank_two_cycle"]
    G, eng = both(tg, g["V"], g["src"], g["dst"], P=P)
    assert np.allclose(eng.pagerank(g["T"], g["d"])[0], g["rank"], rtol=1e-6), g["cite"]
    g = GOLD["bc_undirected_path"]
    G, eng = both(tg, g["V"], g["src"], g["dst"], P=P)
    assert np.allclose(eng.bc(g["sources"])[0], g["bc"], rtol=1e-12), g["cite"]
    if P == 1:
        g = GOLD["pagerank_isolated"]
        G, eng = both(tg, g["V"], g["src"], g["dst"], P=P)
        assert np.allclose(eng.pagerank(g["T"], g["d"])[0], g["rank"], rtol=1e-6), g["cite"]


# ------------------------------------------------------------ C1: RMAT-10, 2 partitions
def test_c1_rmat10_two_partitions(tg):
    scale = 10
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng_dev = tg.Engine.rmat(scale, partitions=2)             # edges generated on the device
    eng_up = tg.Engine.from_edges(V, src, dst, w, partitions=2)  # uploaded host edges
    deg = G.out_degree()
    sources = np.where(deg > 0)[0]
    for eng in (eng_dev, eng_up):
        for s in sources:                       # every source with out-degree >= 1 (8(d) C1)
            assert np.array_equal(eng.bfs(int(s))[0], G.bfs(int(s))), s
        for T in (5, 20):
            assert_pr(eng.pagerank(T)[0], G.pagerank(T))
        for s in sources[::64]:
            assert np.array_equal(eng.sssp(int(s))[0], G.sssp(int(s)))
        bs = inputs.list_sources(src, 4)
        assert_bc(eng.bc(bs)[0], G.bc(bs))


def test_c1_partition_layout_matches_oracle(tg):
    """Structural parity of the partitioner: per-partition |V_p| and the
    source-reduced outbox sizes equal the oracle's degree partition + beta."""
    scale = 10
    src, dst, _ = inputs.rmat_edges(scale)
    V = 1 << scale
    G = oracle.Graph(V, src, dst)
    for P in (2, 3, 4):
        part, _ = G.partition(P)
        br, bd, slots = oracle.beta(V, src, dst, part, P)
        eng = tg.Engine.from_edges(V, src, dst, partitions=P)
        tot_slots = 0
        for p in range(P):
            pi = eng.partition_info(p)
            assert pi["Vp"] == int((part == p).sum())
            assert pi["Ep"] == int((part[src] == p).sum())
            assert pi["Ep_local"] == int(((part[src] == p) & (part[dst] == p)).sum())
            assert np.array_equal(pi["slots_to"], slots[p]), (P, p)
            assert pi["inbox_slots"] == int(slots[:, p].sum())
            tot_slots += pi["outbox_slots"]
        assert np.isclose(tot_slots / len(src), bd)


@pytest.mark.parametrize("P", [2, 3, 8])
def test_random_partitioning_layout_and_parity(tg, P):
    """TG_PART_RANDOM (Fig. 4's "naive random-based" baseline): the
    partition layout (|V_p|, |E_p|, local edges, outbox sizes per peer) equals
    the oracle's random partition + beta, and every algorithm still matches the
    oracle (results do not depend on the partitioning)."""
    scale = 12
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    keys = inputs.part_keys(V)
    part, _ = G.partition_random(P, keys)
    _, _, slots = oracle.beta(V, src, dst, part, P)
    for eng in (tg.Engine.from_edges(V, src, dst, w, partitions=P, strategy=tg.TG_PART_RANDOM),
                tg.Engine.rmat(scale, partitions=P, strategy=tg.TG_PART_RANDOM)):
        assert eng.info["strategy"] == tg.TG_PART_RANDOM
        for p in range(P):
            pi = eng.partition_info(p)
            assert pi["Vp"] == int((part == p).sum())
            assert pi["Ep"] == int((part[src] == p).sum())
            assert pi["Ep_local"] == int(((part[src] == p) & (part[dst] == p)).sum())
            assert np.array_equal(pi["slots_to"], slots[p]), (P, p)
        bs = [int(x) for x in inputs.list_sources(src, 3)]
        check_all(tg, G, eng, bfs_src=bs, sssp_src=bs[:2], pr_T=(5,), bc_src=bs[:2])
        assert np.array_equal(eng.cc()[0], G.cc())
        eng.close()


# ------------------------------------------------------------ partition invariance
@pytest.mark.parametrize("P", [1, 2, 3, 4, 8])
def test_partition_invariance_rmat12(tg, P):
    scale = 12
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.from_edges(V, src, dst, w, partitions=P)
    srcs = inputs.list_sources(src, 6)
    check_all(tg, G, eng, bfs_src=srcs, sssp_src=srcs[:3], pr_T=(5,), bc_src=srcs[:4])


@pytest.mark.parametrize("streams", ["0", "1"])
def test_partition_streams_same_result(tg, streams, monkeypatch):
    """Engine::each_part: the partitions one process hosts launch every phase on
    their own streams (fork / join per phase; TG_PART_STREAMS=1, the default)
    or one after another on one stream (0).  Same oracle results, all five
    algorithms, both transports, forced pull / push directions included."""
    monkeypatch.setenv("TG_PART_STREAMS", streams)
    scale = 12
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    srcs = inputs.list_sources(src, 4)
    cc_ref = G.cc()
    for direction in ("auto", "bottom", "top"):
        monkeypatch.setenv("TG_DIRECTION", direction)
        for mode in ("fused", "copy"):
            eng = tg.Engine.from_edges(V, src, dst, w, partitions=5)
            eng.set_exchange(tg.TG_EXCHANGE_FUSED if mode == "fused" else tg.TG_EXCHANGE_COPY)
            check_all(tg, G, eng, bfs_src=srcs, sssp_src=srcs[:2], pr_T=(5,), bc_src=srcs[:2])
            assert np.array_equal(eng.cc()[0], cc_ref)
            eng.close()


@pytest.mark.parametrize("P", [2, 3, 8])
@pytest.mark.parametrize("mode", ["copy", "fused"])
def test_exchange_modes_rmat13(tg, P, mode):
    """Both communication-phase transports (tg_engine_set_exchange): outbox +
    segment copies, and boundary messages written by the compute kernels
    straight into the receivers' arenas.  Same oracle results either way, for
    all five algorithms, interleaved (each reuses the arenas the previous one
    wrote)."""
    scale = 13
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.from_edges(V, src, dst, w, partitions=P)
    eng.set_exchange(tg.TG_EXCHANGE_FUSED if mode == "fused" else tg.TG_EXCHANGE_COPY)
    srcs = inputs.list_sources(src, 5)
    # twice in a row: arenas left by one run (and by another algorithm) must not leak
    check_all(tg, G, eng, bfs_src=srcs, sssp_src=srcs[:3], pr_T=(5, 6), bc_src=srcs[:2])
    check_all(tg, G, eng, bfs_src=srcs[:2], sssp_src=srcs[:2], pr_T=(1,))
    cc_ref = G.cc()
    for _ in range(2):
        assert np.array_equal(eng.cc()[0], cc_ref), "CC mismatch"
    check_all(tg, G, eng, bfs_src=srcs[:1], pr_T=(), bc_src=srcs[2:4])
    _, st = eng.bfs(int(srcs[0]))
    assert st.comm_bytes > 0


@pytest.mark.parametrize("P", [2, 3, 8])
def test_pagerank_ghost_pull(tg, P):
    """Ghost-pull PageRank (TOTEM_COMM_PULL, tg_engine_set_pagerank_comm):
    boundary sources publish their contributions into the peers' ghost slots
    and every partition pulls over its ghost-indexed in-CSR; same oracle
    result as the push partial sums, repeated and interleaved with push."""
    scale = 13
    src, dst, _ = inputs.rmat_edges(scale)
    V = 1 << scale
    G = oracle.Graph(V, src, dst)
    eng = tg.Engine.from_edges(V, src, dst, partitions=P, weighted=False)
    for T in (1, 5, 6):
        ref = G.pagerank(T)
        eng.set_pagerank_comm(tg.TG_PR_PULL)
        r_pull, st = eng.pagerank(T)
        assert_pr(r_pull, ref)
        assert T == 1 or st.comm_bytes > 0
        eng.set_pagerank_comm(tg.TG_PR_PUSH)
        assert_pr(eng.pagerank(T)[0], ref)
    # a multigraph with self-loops, duplicates and isolated vertices
    rng = np.random.default_rng(8)
    V2 = 400
    s2 = np.concatenate([rng.integers(0, 200, 3000), [5, 5, 7]]).astype(np.uint32)
    d2 = np.concatenate([rng.integers(0, 200, 3000), [5, 9, 9]]).astype(np.uint32)
    G2 = oracle.Graph(V2, s2, d2)
    e2 = tg.Engine.from_edges(V2, s2, d2, partitions=P, weighted=False)
    e2.set_pagerank_comm(tg.TG_PR_PULL)
    assert_pr(e2.pagerank(5)[0], G2.pagerank(5))


@pytest.mark.parametrize("P", [1, 2, 3])
def test_pagerank_hub_split(tg, P, monkeypatch):
    """Hub split (PRHub, TG_PR_HUB=K): the in-edges from the K hub sources of
    the CTA- and warp-class rows are summed by a separate pass from a
    shared-memory replica of the contributions, the class pulls start after
    each row's hub prefix.  Same oracle result for K from 1 to beyond V, in
    both PageRank communications, and for a row whose hub prefix spans several
    tasks (> 4096 hub in-edges)."""
    scale = 13
    src, dst, _ = inputs.rmat_edges(scale)
    V = 1 << scale
    G = oracle.Graph(V, src, dst)
    eng = tg.Engine.from_edges(V, src, dst, partitions=P, weighted=False)
    ref = G.pagerank(5)
    for K in ("1", "256", "3000", "100000", "0"):
        monkeypatch.setenv("TG_PR_HUB", K)
        for comm in ((tg.TG_PR_PUSH, tg.TG_PR_PULL) if P > 1 else (None,)):
            if comm is not None:
                eng.set_pagerank_comm(comm)
            assert_pr(eng.pagerank(5)[0], ref)
    # in-star: 9000 sources of out-degree 1 (ties: all of them lead the
    # out-degree order) point at one row, plus a sparse background
    rng = np.random.default_rng(11)
    n = 10000
    s2 = np.concatenate([np.arange(9000), rng.integers(0, n, 2000)]).astype(np.uint32)
    d2 = np.concatenate([np.full(9000, n - 1), rng.integers(0, n, 2000)]).astype(np.uint32)
    G2 = oracle.Graph(n, s2, d2)
    e2 = tg.Engine.from_edges(n, s2, d2, partitions=P, weighted=False)
    ref2 = G2.pagerank(5)
    for K in ("8192", "5000", "4097"):
        monkeypatch.setenv("TG_PR_HUB", K)
        assert_pr(e2.pagerank(5)[0], ref2)


@pytest.mark.parametrize("P", [1, 2])
def test_pagerank_short_row_groups(tg, P, monkeypatch):
    """TG_PR_GROUP=1: rows of in-degree < 32 summed 32 rows at a time through a
    shared-memory window of 128 in-edges.  Groups whose edges span many
    windows (every row with 31 in-edges: 992 per group), mixed groups holding
    a long row, empty rows and a ragged last group."""
    monkeypatch.setenv("TG_PR_GROUP", "1")
    rng = np.random.default_rng(13)
    n = 2000
    dst = np.repeat(np.arange(n), 31)
    src = rng.integers(0, n, len(dst))
    extra_d = np.full(300, 5)                    # one long row inside a group
    extra_s = rng.integers(0, n, 300)
    sp = np.concatenate([src, extra_s, [7, 7]]).astype(np.uint32)
    dp = np.concatenate([dst, extra_d, [n + 10, n + 40]]).astype(np.uint32)
    V = n + 45                                   # rows n..n+44: 2 edges, mostly empty
    G = oracle.Graph(V, sp, dp)
    eng = tg.Engine.from_edges(V, sp, dp, partitions=P, weighted=False)
    assert_pr(eng.pagerank(5)[0], G.pagerank(5))


@pytest.mark.parametrize("kb", ["8", "15"])
def test_pagerank_cold_tail(tg, kb, monkeypatch):
    """Cold-tail propagation blocking (PRCold, TG_PR_COLD=T): in-edges from the
    sources >= T are summed by the two blocking phases (contributions written
    into per-target-bin slots in source order, then per-bin shared-memory
    sums), the pull gathers only each row's hot prefix and adds the cold sum.
    Same oracle result for T from 1 (every source cold) to beyond the last
    source with out-edges, bins of 2^8 and 2^15 rows; at P = 2 the layout is
    off and the plain pull runs."""
    monkeypatch.setenv("TG_PR_COLD_KB", kb)
    scale = 13
    src, dst, _ = inputs.rmat_edges(scale)
    V = 1 << scale
    G = oracle.Graph(V, src, dst)
    ref = G.pagerank(5)
    for P in (1, 2):
        eng = tg.Engine.from_edges(V, src, dst, partitions=P, weighted=False)
        for T in ("1", "100", "2000", "8000", "100000", "0"):
            monkeypatch.setenv("TG_PR_COLD", T)
            assert_pr(eng.pagerank(5)[0], ref)
            monkeypatch.setenv("TG_PR_GROUP", "1")   # variants fall back to the plain pull
            assert_pr(eng.pagerank(5)[0], ref)
            monkeypatch.delenv("TG_PR_GROUP")
        eng.close()
    rng = np.random.default_rng(14)
    n = 3000
    s2 = np.concatenate([rng.integers(0, n, 20000), [5, 5, 5]]).astype(np.uint32)
    d2 = np.concatenate([rng.integers(0, n, 20000), [5, 6, 6]]).astype(np.uint32)
    G2 = oracle.Graph(n + 7, s2, d2)
    e2 = tg.Engine.from_edges(n + 7, s2, d2, weighted=False)
    for T in ("1", "1500", "2999"):
        monkeypatch.setenv("TG_PR_COLD", T)
        assert_pr(e2.pagerank(5)[0], G2.pagerank(5))


def test_die_map(tg):
    """The measured SM -> die map of a B200: two clusters of pointer-chase
    latency (each die's L2 caches its own SMs' reads), neither tiny."""
    ok, die = tg.tg_device_die_map(0)
    assert len(die) >= 1
    if ok:
        n1 = int(die.sum())
        assert 0 < n1 < len(die) and min(n1, len(die) - n1) * 5 >= len(die)


@pytest.mark.parametrize("P", [1, 2, 3])
def test_pagerank_die_split(tg, P, monkeypatch):
    """Die split (PRSplit, TG_PR_SPLIT=1): every row's in-edges are split into
    two CSRs by the die that gathers the source, each die's SMs pull over
    their own half (stealing from the other die's queue at the end), and a
    finalize pass adds the two partial sums.  Same oracle result as the class
    pulls, in both PageRank communications, including rows cut into chunks
    (> 2048 half-edges)."""
    ok, _ = tg.tg_device_die_map(0)
    if not ok:
        pytest.skip("one-die GPU: no die split")
    monkeypatch.setenv("TG_PR_SPLIT", "1")
    scale = 13
    src, dst, _ = inputs.rmat_edges(scale)
    V = 1 << scale
    G = oracle.Graph(V, src, dst)
    eng = tg.Engine.from_edges(V, src, dst, partitions=P, weighted=False)
    for T in (1, 5):
        ref = G.pagerank(T)
        for comm in ((tg.TG_PR_PUSH, tg.TG_PR_PULL) if P > 1 else (None,)):
            if comm is not None:
                eng.set_pagerank_comm(comm)
            assert_pr(eng.pagerank(T)[0], ref)
    rng = np.random.default_rng(12)
    n = 20000
    s2 = np.concatenate([np.arange(15000), rng.integers(0, n, 4000)]).astype(np.uint32)
    d2 = np.concatenate([np.full(15000, n - 1), rng.integers(0, n, 4000)]).astype(np.uint32)
    G2 = oracle.Graph(n, s2, d2)
    e2 = tg.Engine.from_edges(n, s2, d2, partitions=P, weighted=False)
    assert_pr(e2.pagerank(5)[0], G2.pagerank(5))


def test_set_exchange_rejects_unknown_mode(tg):
    from paper_1312_3018_b200 import tgraph

    eng = tg.Engine.rmat(8, partitions=2)
    with pytest.raises(tgraph.TGraphError) as e:
        eng.set_exchange(7)
    assert e.value.code == tgraph.TG_EINVAL
    with pytest.raises(tgraph.TGraphError) as e:
        eng.set_pagerank_comm(7)
    assert e.value.code == tgraph.TG_EINVAL


@pytest.mark.parametrize("variant", [("TG_PR_SEG", "1"), ("TG_PR_L1", "2"), ("TG_PR_L1", "3"),
                                     ("TG_SSSP_DENSE_DIV", "64"), ("TG_BC_HUBPULL", "0"),
                                     ("TG_BC_HUBPULL", "64"), ("TG_STAGE_ROWOFF", "1"),
                                     ("TG_CC_GHOST_WARP", "1"), ("TG_CC_GHOST_WARP", "0"),
                                     ("TG_PR_REP", "1024"), ("TG_PR_NEXTPOL", "2"),
                                     ("TG_PR_HUB", "512"), ("TG_PR_GROUP", "1"),
                                     ("TG_PR_PIPE", "3"), ("TG_SSSP_CLASS_DIV", "1000000"),
                                     ("TG_PR_PRED", "4,8,4"), ("TG_PR_PRED", "2,6,2"),
                                     ("TG_PR_PRED", "-4,-8,-4"), ("TG_PR_PRED", "0,-4,0"),
                                     ("TG_PR_PRED", "-8,-6,-8"), ("TG_PR_PRED", "0,0,-2"),
                                     ("TG_PR_PRED", "-108,-108,-4"), ("TG_PR_PRED", "-16,-8,-4")])
@pytest.mark.parametrize("P", [1, 3])
def test_kernel_variants_same_result(tg, variant, P, monkeypatch):
    """The A/B kernel variants behind run-time switches
    give the oracle's results too: they only change how the same sums / minima
    are formed."""
    monkeypatch.setenv(*variant)
    scale = 13
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.from_edges(V, src, dst, w, partitions=P)
    srcs = inputs.list_sources(src, 3)
    check_all(tg, G, eng, bfs_src=srcs, sssp_src=srcs[:2], pr_T=(5,), bc_src=srcs[:2])
    assert np.array_equal(eng.cc()[0], G.cc())


@pytest.mark.parametrize("mode", ["top", "bottom", "auto"])
@pytest.mark.parametrize("P", [1, 2, 3, 8])
def test_direction_modes_same_result(tg, mode, P, monkeypatch):
    """Direction-optimizing BFS / pull-sigma BC: top-down,
    forced bottom-up and the automatic switch all give the oracle's result, on
    one partition and across P partitions (P > 1: the pulls read remote
    in-neighbours through ghost frontier bits / sigma published by their
    owners), in both exchange transports."""
    monkeypatch.setenv("TG_DIRECTION", mode)
    scale = 13
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.from_edges(V, src, dst, w, partitions=P)
    srcs = inputs.list_sources(src, 5)
    for x in ((tg.TG_EXCHANGE_FUSED, tg.TG_EXCHANGE_COPY) if P > 1 else (None,)):
        if x is not None:
            eng.set_exchange(x)
        for s in srcs:
            assert np.array_equal(eng.bfs(int(s))[0], G.bfs(int(s))), (mode, s)
        assert_bc(eng.bc(srcs[:3])[0], G.bc(srcs[:3]))
    # a path: every level is tiny, bottom-up must still be exact
    n = 500
    p_src = np.arange(n - 1, dtype=np.uint32)
    Gp, ep = both(tg, n, p_src, p_src + 1, P=P)
    assert np.array_equal(ep.bfs(0)[0], Gp.bfs(0))
    assert_bc(ep.bc([0, 3])[0], Gp.bc([0, 3]))


# ------------------------------------------------------------ adversarial shapes
@pytest.mark.parametrize("P", [1, 2])
def test_hub_of_degree_2_20(tg, P):
    k = 1 << 20
    V = k + 2
    src = np.concatenate([np.zeros(k, np.uint32), np.arange(1, 200, dtype=np.uint32)])
    dst = np.concatenate([np.arange(1, k + 1, dtype=np.uint32), np.full(199, k + 1, np.uint32)])
    w = (np.arange(len(src)) % 63 + 1).astype(np.uint32)
    G, eng = both(tg, V, src, dst, w, P)
    check_all(tg, G, eng, bfs_src=[0, 5], sssp_src=[0], pr_T=(3,), bc_src=[0, 7])


@pytest.mark.parametrize("P", [1, 3])
def test_long_path_many_supersteps(tg, P):
    n = 3000
    src = np.arange(n - 1, dtype=np.uint32)
    dst = src + 1
    w = np.full(n - 1, 63, np.uint32)
    G, eng = both(tg, n, src, dst, w, P)
    lv, st = eng.bfs(0)
    assert st.supersteps == n and np.array_equal(lv, G.bfs(0))
    check_all(tg, G, eng, sssp_src=[0, 1500], pr_T=(4,), bc_src=[0, 10])


@pytest.mark.parametrize("P", [1, 2])
def test_multigraph_selfloops_disconnected_isolated(tg, P):
    rng = np.random.default_rng(11)
    n = 5000
    src = rng.integers(0, n // 2, 40000).astype(np.uint32)   # upper half: isolated vertices
    dst = rng.integers(0, n // 2, 40000).astype(np.uint32)
    src = np.concatenate([src, src[:5000], np.arange(100, dtype=np.uint32)])  # duplicates
    dst = np.concatenate([dst, dst[:5000], np.arange(100, dtype=np.uint32)])  # + self loops
    w = rng.integers(1, 64, len(src)).astype(np.uint32)
    G, eng = both(tg, n, src, dst, w, P)
    check_all(tg, G, eng, bfs_src=[0, 3, n - 1], sssp_src=[0, n - 1], pr_T=(5,),
              bc_src=[0, 1, n - 1])


def test_uniform_degree_cycle_and_empty_graph(tg):
    n = 10007
    src = np.arange(n, dtype=np.uint32)
    dst = ((src.astype(np.int64) * 7 + 1) % n).astype(np.uint32)
    G, eng = both(tg, n, src, dst, np.ones(n, np.uint32), 2)
    check_all(tg, G, eng, bfs_src=[0], sssp_src=[5], pr_T=(5,), bc_src=[0])
    G, eng = both(tg, 7, [], [], None, 1)
    lv, _ = eng.bfs(3)
    assert lv.tolist() == [0xFFFFFFFF] * 3 + [0] + [0xFFFFFFFF] * 3
    r, _ = eng.pagerank(2)
    assert np.allclose(r, 0.15 / 7, rtol=1e-6)


def test_errors(tg):
    src, dst, _ = inputs.rmat_edges(8)
    eng = tg.Engine.from_edges(256, src, dst)
    with pytest.raises(tg.TGraphError) as e:
        eng.bfs(256)                       # source >= V
    assert e.value.code == 2
    with pytest.raises(tg.TGraphError) as e:
        eng.sssp(0)                        # unweighted engine
    assert e.value.code == 2
    with pytest.raises(tg.TGraphError) as e:
        eng.pagerank(0)                    # iterations < 1
    assert e.value.code == 2
    with pytest.raises(tg.TGraphError):
        tg.Engine.from_edges(10, [0, 11], [1, 2])  # id >= V


def test_device_outputs(tg):
    import torch

    scale = 10
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.rmat(scale)
    s = int(inputs.rmat_sources(scale, 1)[0])
    lv = torch.empty(V, dtype=torch.int32, device="cuda")
    eng.bfs(s, out=lv)
    assert np.array_equal(lv.cpu().numpy().view(np.uint32), G.bfs(s))
    r = torch.empty(V, dtype=torch.float32, device="cuda")
    eng.pagerank(5, out=r)
    assert_pr(r.cpu().numpy(), G.pagerank(5))


def layered(width, layers):
    """Source 0 -> layer 1 -> ... -> layer `layers`, complete bipartite between
    consecutive layers: sigma at layer k = width^(k-1) (width^k paths minus the
    single source fan-out)."""
    src, dst = [], []
    prev = [0]
    nxt_id = 1
    for _ in range(layers):
        cur = list(range(nxt_id, nxt_id + width))
        nxt_id += width
        for a in prev:
            for b in cur:
                src.append(a)
                dst.append(b)
        prev = cur
    return nxt_id, np.array(src, np.uint32), np.array(dst, np.uint32)


def test_bc_sigma_exactness_guard(tg):
    # reading A11: sigma is an fp64 path count, exact below 2^53.  Width 2,
    # 53 layers: sigma tops out at 2^52 -> exact, equals the oracle; width 2,
    # 55 layers: 2^54 -> TG_EINTERNAL instead of a silently rounded answer.
    V, s, d = layered(2, 53)
    G, eng = both(tg, V, s, d)
    assert_bc(eng.bc([0])[0], G.bc([0]))
    V, s, d = layered(2, 55)
    eng = tg.Engine.from_edges(V, s, d)
    with pytest.raises(tg.TGraphError) as e:
        eng.bc([0])
    assert e.value.code == 5 and "2^53" in str(e.value)


# ------------------------------------------------- host graphs / input generation
def test_rmat_slice_matches_the_generator(tg):
    # tg_rmat_edges (device) and inputs.rmat_edges (host C) evaluate the same
    # counter-based stream: any slice agrees element by element.
    for scale, first, count in ((12, 0, 5000), (20, 123456789 % (16 << 20), 70000)):
        s, d, w = tg.tg_rmat_edges(scale, first=first, count=count, weights=True)
        hs, hd, hw = inputs.rmat_edges(scale, first=first, count=count, weights=True)
        assert np.array_equal(s, hs) and np.array_equal(d, hd) and np.array_equal(w, hw)
    import torch
    out = tuple(torch.empty(3000, dtype=torch.int32, device="cuda:0") for _ in range(3))
    tg.tg_rmat_edges(10, a=0.25, b=0.25, c=0.25, first=77, count=3000, out=out, weights=True)
    hs, hd, hw = inputs.rmat_edges(10, a=0.25, b=0.25, c=0.25, first=77, count=3000, weights=True)
    for t, h in zip(out, (hs, hd, hw)):
        assert np.array_equal(t.cpu().numpy().view(np.uint32), h)


@pytest.mark.parametrize("P", [1, 3])
def test_engine_from_edge_list_file(tg, tmp_path, P):
    rng = np.random.default_rng(11)
    V, E = 300, 2400
    src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
    w = rng.integers(1, 64, E)
    path = tmp_path / "g.txt"
    with open(path, "w") as f:
        f.write(f"# nodes: {V}\n")
        for a, b, c in zip(src, dst, w):
            f.write(f"{a} {b} {c}\n")
    g = tg.Graph.load_edge_list(str(path), weighted=True)
    eng = tg.Engine.from_graph(g, partitions=P)
    G = oracle.Graph(V, src, dst, w)
    check_all(tg, G, eng, bfs_src=(0, 5, 299), sssp_src=(0, 17), pr_T=(1, 5), bc_src=(0, 3, 8))


def test_uniform_graph(tg):
    # (a, b, c) = (0.25, 0.25, 0.25): every endpoint bit fair -- the UNIFORM
    # graph of the paper's Fig. 4 / SPEC generate_uniform
    scale = 12
    src, dst, w = inputs.rmat_edges(scale, a=0.25, b=0.25, c=0.25, weights=True)
    G = oracle.Graph(1 << scale, src, dst, w)
    for P in (1, 4):
        eng = tg.Engine.rmat(scale, a=0.25, b=0.25, c=0.25, partitions=P)
        ss = inputs.rmat_sources(scale, 3, a=0.25, b=0.25, c=0.25)
        check_all(tg, G, eng, bfs_src=ss, sssp_src=ss[:2], pr_T=(5,), bc_src=ss[:2])


# ------------------------------------------------------------ C2: RMAT-22, 1 GPU
@pytest.fixture(scope="module")
def c2(tg):
    scale = 22
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    G = oracle.Graph(1 << scale, src, dst, w)
    del src, dst, w
    eng = tg.Engine.rmat(scale)          # device-side generation of the same stream
    return scale, G, eng


def test_c2_bfs_sssp(c2):
    """BFS x 64 and SSSP x 64 sources, every one bit-exact
    against the full oracle (oracle runs in forked children, one per core)."""
    from forkpool import fork_map

    scale, G, eng = c2
    srcs = [int(s) for s in inputs.rmat_sources(scale, 64)]
    deg = G.out_degree()
    lvs, dists = [], []
    for s in srcs:
        lv, st = eng.bfs(s)
        assert st.traversed_edges == int(deg[lv != 0xFFFFFFFF].sum())
        lvs.append(lv.copy())
        dists.append(eng.sssp(s)[0].copy())
    jobs = [(lambda i=i: bool(np.array_equal(lvs[i], G.bfs(srcs[i])))) for i in range(64)]
    jobs += [(lambda i=i: bool(np.array_equal(dists[i], G.sssp(srcs[i])))) for i in range(64)]
    ok = fork_map(jobs)
    bad = [("bfs" if j < 64 else "sssp", srcs[j % 64]) for j, o in enumerate(ok) if not o]
    assert not bad, bad


def test_c2_pagerank_bc(c2):
    scale, G, eng = c2
    assert_pr(eng.pagerank(5)[0], G.pagerank(5))
    bs = inputs.rmat_sources(scale, 2)
    assert_bc(eng.bc(bs)[0], G.bc(bs))


# ------------------------------------------------------------ C3: RMAT-26, 1/2/4 partitions
@pytest.mark.slow
def test_c3_rmat26_pagerank_bc_partitions(tg):
    """BASELINE configs[2]: RMAT-26, PageRank (T = 5) and BC from sampled
    sources over 1, 2 and 4 degree-aware partitions (one B200 hosts all of
    them here; the multi-process path is the same partition code), full oracle.
    Fused exchange by default; PageRank at P = 4 also through the copy path
    and with ghost-pull communication.  BC: k = 4 sources,
    each checked on its own against its own Brandes run (the four oracle runs
    side by side in forked children)."""
    from forkpool import fork_map

    scale = 26
    srcs = [int(x) for x in inputs.rmat_sources(scale, 4)]
    prs, bcs = [], []
    for P in (1, 2, 4):
        eng = tg.Engine.rmat(scale, partitions=P, weighted=False)
        prs.append(eng.pagerank(5)[0].copy())
        if P == 4:
            eng.set_exchange(tg.TG_EXCHANGE_COPY)
            prs.append(eng.pagerank(5)[0].copy())
            eng.set_exchange(tg.TG_EXCHANGE_FUSED)
            eng.set_pagerank_comm(tg.TG_PR_PULL)   # ghost-pull at scale
            prs.append(eng.pagerank(5)[0].copy())
            eng.set_pagerank_comm(tg.TG_PR_PUSH)
        bcs.append([eng.bc([x])[0].copy() for x in srcs])
        eng.close()
    src, dst, _ = inputs.rmat_edges(scale)
    G = oracle.Graph(1 << scale, src, dst)
    del src, dst

    def pr_job():  # oracle PageRank and BC side by side (forked children)
        ref = G.pagerank(5)
        return max(float((np.abs(g.astype(np.float64) - ref) / np.abs(ref)).max()) for g in prs)

    def bc_job(i):
        ref = G.bc([srcs[i]])
        scale_ = max(1.0, float(np.abs(ref).max()))
        return max(int((np.abs(run[i] - ref) > BC_RTOL * np.abs(ref) + 1e-12 * scale_).sum())
                   for run in bcs)

    res = fork_map([pr_job] + [functools.partial(bc_job, i) for i in range(len(srcs))])
    pr_err, bc_bad = res[0], res[1:]
    assert pr_err <= PR_RTOL, f"PageRank max rel err {pr_err:.3e}"
    assert not any(bc_bad), f"BC: vertices outside the bar per source {bc_bad}"


@pytest.mark.parametrize("P", [1, 3])
def test_sssp_wide_weights_and_overflow(tg, P):
    """Weights >= 256 keep the 4-byte weight array (the byte form is used only
    when every weight fits); a distance past 2^32 - 1 is TG_EINTERNAL (reading
    A18), not a wrapped value."""
    from paper_1312_3018_b200 import tgraph

    rng = np.random.default_rng(21)
    V, E = 600, 5000
    src, dst = rng.integers(0, V, E), rng.integers(0, V, E)
    w = rng.integers(1, 1 << 20, E)
    G, eng = both(tg, V, src, dst, w, P=P)
    for s in (0, 7, 311):
        assert np.array_equal(eng.sssp(s)[0], G.sssp(s)), s
    # 0 -> 1 -> 2 with weights 2^31 each: dist(2) = 2^32 does not fit u32
    eng2 = tg.Engine.from_edges(3, np.array([0, 1], np.uint32), np.array([1, 2], np.uint32),
                                np.array([1 << 31, 1 << 31], np.uint32), partitions=P)
    with pytest.raises(tgraph.TGraphError) as e:
        eng2.sssp(0)
    assert e.value.code == tgraph.TG_EINTERNAL


def test_async_host_collection(tg):
    """tg_engine_set_async_collect: host outputs of consecutive calls (copied
    on the library's copy stream while the next algorithm runs, two staging
    buffers in rotation) are all exact once tg_engine_sync returns; off again,
    outputs are complete on return."""
    scale = 14
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    eng = tg.Engine.from_edges(V, src, dst, w)
    srcs = [int(x) for x in inputs.list_sources(src, 3)]
    eng.set_async_collect(True)
    outs = []
    for s in srcs:
        lv, ds = np.empty(V, np.uint32), np.empty(V, np.uint32)
        b, pr = np.empty(V), np.empty(V, np.float32)
        eng.bc([s], out=b)
        eng.bfs(s, out=lv)
        eng.pagerank(5, out=pr)
        eng.sssp(s, out=ds)
        outs.append((s, lv, ds, pr, b))
    eng.sync()
    ref_pr = G.pagerank(5)
    for s, lv, ds, pr, b in outs:
        assert np.array_equal(lv, G.bfs(s)) and np.array_equal(ds, G.sssp(s))
        assert_pr(pr, ref_pr)
        assert_bc(b, G.bc([s]))
    # collection tickets: double buffering -- after each round of four calls,
    # the previous round's ticket is waited on and its outputs are exact while
    # this round's copies may still be in flight; more rounds than ticket slots
    t0 = eng.last_ticket()
    assert t0 == 4 * len(srcs)
    sets = [(np.empty(V, np.uint32), np.empty(V)) for _ in range(2)]
    prev = t0
    for k in range(20):
        s = srcs[k % len(srcs)]
        lv, b = sets[k % 2]
        eng.bc([s], out=b)
        eng.bfs(s, out=lv)
        eng.wait_ticket(prev)
        if k:
            s0 = srcs[(k - 1) % len(srcs)]
            lv0, b0 = sets[(k - 1) % 2]
            assert np.array_equal(lv0, G.bfs(s0))
            assert_bc(b0, G.bc([s0]))
        prev = eng.last_ticket()
        assert prev == t0 + 2 * (k + 1)
    eng.wait_ticket(prev)
    assert np.array_equal(sets[19 % 2][0], G.bfs(srcs[19 % len(srcs)]))
    with pytest.raises(tg.TGraphError):
        eng.wait_ticket(prev + 1)
    eng.wait_ticket(0)
    eng.set_async_collect(False)
    assert np.array_equal(eng.bfs(srcs[0])[0], G.bfs(srcs[0]))
    eng.close()


def test_in_csr_only_engine(tg):
    """build_in_csr = 2 (the out-CSR released after the build): PageRank matches
    the oracle at P = 1; the frontier algorithms refuse with TG_EINVAL."""
    scale = 12
    src, dst, _ = inputs.rmat_edges(scale)
    V = 1 << scale
    G = oracle.Graph(V, src, dst)
    eng = tg.Engine.from_edges(V, src, dst, in_csr=2)
    assert_pr(eng.pagerank(5)[0], G.pagerank(5))
    for call in (lambda: eng.bfs(0), lambda: eng.sssp(0), lambda: eng.bc([0]), lambda: eng.cc()):
        with pytest.raises(tg.TGraphError) as e:
            call()
        assert e.value.code == tg.tgraph.TG_EINVAL
    full = tg.Engine.from_edges(V, src, dst)
    assert eng.info["device_bytes"] < full.info["device_bytes"]
    eng.close()
    full.close()
    # several partitions: each partition's out-CSR is dropped as soon as its
    # in-CSR and inbox are built
    for P in (2, 3):
        part = tg.Engine.from_edges(V, src, dst, in_csr=2, partitions=P)
        assert_pr(part.pagerank(5)[0], G.pagerank(5))
        part.close()
    # device-generated edges: the in-CSR is filled from the edge stream (no
    # out-CSR columns at all); multigraph with self-loops and isolated vertices
    gen = tg.Engine.rmat(scale, weighted=False, in_csr=2)
    assert_pr(gen.pagerank(5)[0], G.pagerank(5))
    gen.close()
    rng = np.random.default_rng(15)
    s2 = np.concatenate([rng.integers(0, 300, 5000), [7, 7, 9]]).astype(np.uint32)
    d2 = np.concatenate([rng.integers(0, 300, 5000), [7, 8, 8]]).astype(np.uint32)
    G2 = oracle.Graph(400, s2, d2)
    e2 = tg.Engine.from_edges(400, s2, d2, in_csr=2)
    assert_pr(e2.pagerank(20)[0], G2.pagerank(20))
    e2.close()


@pytest.mark.parametrize("skip", ["1", "0"])
def test_pagerank_sink_rows_stats(tg, skip, monkeypatch):
    """Non-final PageRank rounds do not pull the rows of sinks (out-degree 0;
    their intermediate ranks feed no output, TG_PR_SINKSKIP): ranks equal the
    oracle's either way, and the stats count only the edges pulled --
    E x T minus the sinks' in-edges in the T - 1 non-final rounds."""
    monkeypatch.setenv("TG_PR_SINKSKIP", skip)
    scale, T = 12, 5
    src, dst, _ = inputs.rmat_edges(scale)
    V, E = 1 << scale, len(src)
    G = oracle.Graph(V, src, dst)
    into_sinks = int((np.bincount(src, minlength=V)[dst] == 0).sum())
    assert 0 < into_sinks < E // 20
    for P in (1, 3):
        eng = tg.Engine.from_edges(V, src, dst, partitions=P)
        r, st = eng.pagerank(T)
        assert_pr(r, G.pagerank(T))
        want = E * T - (into_sinks * (T - 1) if skip == "1" and P == 1 else 0)
        assert st.traversed_edges == want, (P, st.traversed_edges, want)
        eng.close()


@pytest.mark.parametrize("P", [1, 3])
def test_traversed_edge_counts(tg, P):
    """TEPS bases (reading A14): BFS counts the out-degrees of the reached
    vertices, BC twice that (forward + backward), taken from the
    frontiers' exact degree sums -- equal to the oracle's reached set, in every
    direction mode."""
    scale = 12
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    G = oracle.Graph(V, src, dst, w)
    deg = G.out_degree()
    eng = tg.Engine.from_edges(V, src, dst, w, partitions=P)
    for s in inputs.list_sources(src, 3):
        s = int(s)
        want = int(deg[G.bfs(s) != 0xFFFFFFFF].sum())
        assert eng.bfs(s)[1].traversed_edges == want
        assert eng.bc([s])[1].traversed_edges == 2 * want
    eng.close()
