"""Pins for the CPU oracle (oracle/oracle.c), independent of it.

Every oracle function is checked against something other than itself:
exhaustive enumeration, boolean matrix powers, Floyd-Warshall, all-simple-path
enumeration, closed forms, invariants and the worked examples printed in
SPEC.md (tests/golden/spec_examples.json).  Chosen so that a dropped term, a
wrong sign/index or a transposed operand fails at least one of them.
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import INF32

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def edges_of(adj):
    """Multigraph adjacency count matrix -> (src, dst) lists (row-major order)."""
    src, dst = [], []
    n = adj.shape[0]
    for u in range(n):
        for v in range(n):
            for _ in range(int(adj[u, v])):
                src.append(u)
                dst.append(v)
    return np.array(src, np.uint32), np.array(dst, np.uint32)


def random_multigraph(rng, n, m, self_loops=True):
    src = rng.integers(0, n, m).astype(np.uint32)
    dst = rng.integers(0, n, m).astype(np.uint32)
    if not self_loops:
        keep = src != dst
        src, dst = src[keep], dst[keep]
    return src, dst


# ---------------------------------------------------------------- CSR
def test_csr_golden():
    for key in ("csr_path", "csr_empty"):
        g = GOLD[key]
        G = oracle.Graph(g["V"], g["src"], g["dst"])
        assert list(G.row_off) == g["row_off"], g["cite"]
    g = GOLD["csr_weights"]
    G = oracle.Graph(g["V"], g["src"], g["dst"], g["w"])
    assert list(G.col[:2]) == g["col"] and list(G.w[:2]) == g["wout"], g["cite"]


def test_csr_random_multiset():
    rng = np.random.default_rng(0)
    src, dst = random_multigraph(rng, 50, 400)
    G = oracle.Graph(50, src, dst)
    for u in range(50):
        got = sorted(G.col[G.row_off[u]:G.row_off[u + 1]].tolist())
        assert got == sorted(dst[src == u].tolist())


# ------------------------------------------------------------------- BFS
def bfs_by_matrix_powers(A, s):
    """level(v) = min k such that (A^k)[s, v] != 0 (boolean powers)."""
    n = A.shape[0]
    level = np.full(n, INF32, np.uint64)
    reach = np.zeros(n, bool)
    reach[s] = True
    level[s] = 0
    cur = reach.copy()
    for k in range(1, n + 1):
        cur = (cur.astype(int) @ (A > 0).astype(int)) > 0
        newly = cur & ~reach
        level[newly] = k
        reach |= cur
    return level


def test_bfs_exhaustive_n3():
    # every directed graph on 3 vertices incl. self-loops (2^9), every source
    for bits in range(1 << 9):
        A = np.array([(bits >> i) & 1 for i in range(9)]).reshape(3, 3)
        src, dst = edges_of(A)
        G = oracle.Graph(3, src, dst)
        for s in range(3):
            assert np.array_equal(G.bfs(s), bfs_by_matrix_powers(A, s).astype(np.uint32))


def test_bfs_random_n4_multigraphs():
    rng = np.random.default_rng(1)
    for _ in range(1500):
        A = rng.integers(0, 3, (4, 4)) * (rng.random((4, 4)) < 0.4)
        src, dst = edges_of(A)
        G = oracle.Graph(4, src, dst)
        s = int(rng.integers(0, 4))
        assert np.array_equal(G.bfs(s), bfs_by_matrix_powers(A, s).astype(np.uint32))


def floyd_warshall(n, src, dst, w):
    D = np.full((n, n), np.inf)
    np.fill_diagonal(D, 0)
    for u, v, x in zip(src, dst, w):
        D[u, v] = min(D[u, v], x)
    for k in range(n):
        D = np.minimum(D, D[:, [k]] + D[[k], :])
    return D


def test_bfs_and_sssp_vs_floyd_warshall():
    rng = np.random.default_rng(2)
    for trial in range(60):
        n = int(rng.integers(1, 64))
        m = int(rng.integers(0, 4 * n))
        src, dst = random_multigraph(rng, n, m)
        w = rng.integers(1, 64, len(src)).astype(np.uint32)
        G = oracle.Graph(n, src, dst, w)
        Dh = floyd_warshall(n, src, dst, np.ones(len(src)))
        Dw = floyd_warshall(n, src, dst, w.astype(float))
        for s in range(0, n, max(1, n // 5)):
            exp_h = np.where(np.isinf(Dh[s]), INF32, Dh[s]).astype(np.uint64)
            exp_w = np.where(np.isinf(Dw[s]), INF32, Dw[s]).astype(np.uint64)
            assert np.array_equal(G.bfs(s).astype(np.uint64), exp_h)
            assert np.array_equal(G.sssp(s).astype(np.uint64), exp_w)


def test_bfs_sssp_golden():
    for key in ("bfs_path_split", "bfs_isolated_source"):
        g = GOLD[key]
        G = oracle.Graph(g["V"], g["src"], g["dst"])
        assert G.bfs(g["source"]).tolist() == g["levels"], g["cite"]
    g = GOLD["sssp_triangle"]
    G = oracle.Graph(g["V"], g["src"], g["dst"], g["w"])
    assert G.sssp(g["source"]).tolist() == g["dist"], g["cite"]


def test_sssp_unit_weights_equal_bfs_and_scaling():
    # special cases: w == 1 reduces Dijkstra to BFS; w == c scales distances by c
    rng = np.random.default_rng(3)
    src, dst = random_multigraph(rng, 300, 1500)
    G1 = oracle.Graph(300, src, dst, np.ones(len(src), np.uint32))
    G7 = oracle.Graph(300, src, dst, np.full(len(src), 7, np.uint32))
    for s in (0, 17, 123):
        b = G1.bfs(s)
        assert np.array_equal(G1.sssp(s), b)
        exp = np.where(b == INF32, INF32, b.astype(np.uint64) * 7).astype(np.uint32)
        assert np.array_equal(G7.sssp(s), exp)


def test_certificates_accept_truth_reject_perturbations():
    rng = np.random.default_rng(4)
    src, dst = random_multigraph(rng, 200, 1200)
    w = rng.integers(1, 64, len(src)).astype(np.uint32)
    G = oracle.Graph(200, src, dst, w)
    for s in (0, 5):
        lv, d = G.bfs(s), G.sssp(s)
        assert G.bfs_certify(s, lv) and G.sssp_certify(s, d)
        reached = np.where((lv != INF32) & (np.arange(200) != s))[0]
        for v in reached[:10]:
            for delta in (-1, 1):
                bad = lv.copy(); bad[v] = int(lv[v]) + delta
                assert not G.bfs_certify(s, bad)
                badd = d.copy(); badd[v] = int(d[v]) + delta
                assert not G.sssp_certify(s, badd)
            bad = lv.copy(); bad[v] = INF32
            assert not G.bfs_certify(s, bad)


def _raised_tight(G_src, G_dst, G_w, truth, v):
    """The largest value of truth[u] + w over v's reached in-edges: a value for v
    that still has a tight in-edge (certificate condition 3 holds) but is longer
    than the shortest path, so only condition 2 ("no edge has val[u] + w <
    val[v]") can reject it."""
    m = (G_dst == v) & (truth[G_src] != INF32)
    return int((truth[G_src[m]].astype(np.uint64) + G_w[m]).max()) if m.any() else None


def test_certificates_reject_longer_tight_paths():
    """Hand-worked: s->a (1), a->v (1), s->b (5), b->v (1).  dist[v] = 6 is tight
    via b, so the tightness condition alone accepts it; the relaxation condition
    (a->v gives 2 < 6) must reject it.  BFS analog: s->v, s->a, a->v with
    level[v] = 2 (tight via a; the edge s->v gives 1 < 2).  Then the same raise
    on random graphs, in-memory and streaming."""
    s, a, b, v = 0, 1, 2, 3
    src = np.array([s, a, s, b], np.uint32)
    dst = np.array([a, v, b, v], np.uint32)
    w = np.array([1, 1, 5, 1], np.uint32)
    G = oracle.Graph(4, src, dst, w)
    d = G.sssp(s)
    assert list(d) == [0, 1, 5, 2]
    assert G.sssp_certify(s, d)
    bad = d.copy(); bad[v] = 6
    assert not G.sssp_certify(s, bad)
    cert = oracle.StreamingCertificate(4, s, bad, True)
    cert.feed(src, dst, w)
    assert not cert.holds()
    bsrc = np.array([s, s, a], np.uint32)
    bdst = np.array([v, a, v], np.uint32)
    GB = oracle.Graph(4, bsrc, bdst)
    lv = GB.bfs(s)
    assert list(lv) == [0, 1, INF32, 1]
    badl = lv.copy(); badl[v] = 2
    assert not GB.bfs_certify(s, badl)
    cert = oracle.StreamingCertificate(4, s, badl, False)
    cert.feed(bsrc, bdst, np.ones(3, np.uint32))
    assert not cert.holds()

    rng = np.random.default_rng(12)
    n = 400
    src, dst = random_multigraph(rng, n, 3000)
    w = rng.integers(1, 64, len(src)).astype(np.uint32)
    G = oracle.Graph(n, src, dst, w)
    ones = np.ones(len(src), np.uint32)
    raised = 0
    for s in (0, 9, 77):
        for weighted, truth, ww in ((True, G.sssp(s), w), (False, G.bfs(s), ones)):
            for v in np.where((truth != INF32) & (np.arange(n) != s))[0][:40]:
                t = _raised_tight(src, dst, ww, truth, v)
                if t is None or t <= int(truth[v]):
                    continue
                bad = truth.copy(); bad[v] = t
                raised += 1
                inmem = G.sssp_certify(s, bad) if weighted else G.bfs_certify(s, bad)
                assert not inmem
                cert = oracle.StreamingCertificate(n, s, bad, weighted)
                cert.feed(src, dst, ww)
                assert not cert.holds()
    assert raised > 50


# ------------------------------------------------------------------- PageRank
D = 0.85


def test_pagerank_golden():
    for key in ("pagerank_isolated", "pagerank_two_cycle"):
        g = GOLD[key]
        G = oracle.Graph(g["V"], g["src"], g["dst"])
        assert np.allclose(G.pagerank(g["T"], g["d"]), g["rank"], rtol=1e-14), g["cite"]


def test_pagerank_cycle_and_complete_stay_uniform():
    for n in (3, 7, 16):
        cyc = oracle.Graph(n, np.arange(n), (np.arange(n) + 1) % n)
        pairs = [(u, v) for u in range(n) for v in range(n) if u != v]
        K = oracle.Graph(n, [p[0] for p in pairs], [p[1] for p in pairs])
        for T in (1, 5, 20):
            assert np.allclose(cyc.pagerank(T), 1.0 / n, rtol=1e-13)
            assert np.allclose(K.pagerank(T), 1.0 / n, rtol=1e-13)


def test_pagerank_in_star_closed_form():
    # leaves -> center; center dangling.  After T >= 2: leaves (1-d)/n,
    # center (1-d)/n * (1 + d k).  After T = 1: center (1-d)/n + d k / n.
    k = 9
    n = k + 1
    G = oracle.Graph(n, np.arange(1, n), np.zeros(k, np.uint32))
    r1 = G.pagerank(1)
    assert np.isclose(r1[0], (1 - D) / n + D * k / n, rtol=1e-14)
    for T in (2, 3, 6):
        r = G.pagerank(T)
        assert np.allclose(r[1:], (1 - D) / n, rtol=1e-14)
        assert np.isclose(r[0], (1 - D) / n * (1 + D * k), rtol=1e-14)


def test_pagerank_undirected_star_recursion_and_fixed_point():
    # center <-> k leaves: c' = (1-d)/n + d*k*l, l' = (1-d)/n + d*c/k
    k = 6
    n = k + 1
    src = np.concatenate([np.zeros(k), np.arange(1, n)]).astype(np.uint32)
    dst = np.concatenate([np.arange(1, n), np.zeros(k)]).astype(np.uint32)
    G = oracle.Graph(n, src, dst)
    c = l = 1.0 / n
    for T in range(1, 8):
        c, l = (1 - D) / n + D * k * l, (1 - D) / n + D * c / k
        r = G.pagerank(T)
        assert np.isclose(r[0], c, rtol=1e-13) and np.allclose(r[1:], l, rtol=1e-13)
    r = G.pagerank(400)
    assert np.isclose(r[0], (1 + D * k) / (n * (1 + D)), rtol=1e-10)
    assert np.allclose(r[1:], (k + D) / (k * n * (1 + D)), rtol=1e-10)


def test_pagerank_dense_matrix_recurrence_and_mass():
    rng = np.random.default_rng(5)
    for trial in range(30):
        n = int(rng.integers(2, 40))
        src, dst = random_multigraph(rng, n, int(rng.integers(1, 5 * n)))
        G = oracle.Graph(n, src, dst)
        A = np.zeros((n, n))
        np.add.at(A, (dst, src), 1.0)           # A[v, u] = multiplicity of u->v
        out = A.sum(axis=0)
        M = np.divide(A, out, out=np.zeros_like(A), where=out > 0)
        r = np.full(n, 1.0 / n)
        for T in range(1, 6):
            r = (1 - D) / n + D * (M @ r)
            assert np.allclose(G.pagerank(T), r, rtol=1e-12, atol=0)
        if (out > 0).all():                     # dangling-free: mass conserved
            assert abs(G.pagerank(7).sum() - 1.0) < 1e-12


# ------------------------------------------------------------------- BC
def bc_by_path_enumeration(n, src, dst, sources):
    """Enumerate every simple path (as an edge sequence) from each s, keep the
    shortest per target, and sum sigma_st(v)/sigma_st over t != s, v != s,t."""
    adj = [[] for _ in range(n)]
    for u, v in zip(src, dst):
        adj[int(u)].append(int(v))
    bc = np.zeros(n)
    for s in sources:
        paths = {t: [] for t in range(n)}

        def dfs(u, visited, seq):
            for v in adj[u]:
                if v in visited:
                    continue
                paths[v].append(seq + [v])
                dfs(v, visited | {v}, seq + [v])

        dfs(s, {s}, [s])
        for t in range(n):
            if t == s or not paths[t]:
                continue
            L = min(len(p) for p in paths[t])
            short = [p for p in paths[t] if len(p) == L]
            for v in range(n):
                if v in (s, t):
                    continue
                bc[v] += sum(1 for p in short if v in p) / len(short)
    return bc


def test_bc_vs_path_enumeration():
    rng = np.random.default_rng(6)
    for trial in range(80):
        n = int(rng.integers(2, 7))
        src, dst = random_multigraph(rng, n, int(rng.integers(0, 3 * n)), self_loops=False)
        sources = list(range(n)) if trial % 2 else [int(rng.integers(0, n))]
        G = oracle.Graph(n, src, dst)
        assert np.allclose(G.bc(sources), bc_by_path_enumeration(n, src, dst, sources),
                           rtol=1e-12, atol=1e-12)


def test_bc_closed_forms():
    g = GOLD["bc_undirected_path"]
    assert np.allclose(oracle.Graph(g["V"], g["src"], g["dst"]).bc(g["sources"]), g["bc"]), g["cite"]
    for n in (2, 5, 9):
        i = np.arange(n)
        fwd = oracle.Graph(n, i[:-1], i[1:])                          # directed path
        assert np.allclose(fwd.bc(range(n)), i * (n - 1 - i))
        und = oracle.Graph(n, np.r_[i[:-1], i[1:]], np.r_[i[1:], i[:-1]])
        assert np.allclose(und.bc(range(n)), 2 * i * (n - 1 - i))
    k = 5
    star = oracle.Graph(k + 1, np.r_[np.zeros(k), np.arange(1, k + 1)],
                        np.r_[np.arange(1, k + 1), np.zeros(k)])
    r = star.bc(range(k + 1))
    assert np.isclose(r[0], k * (k - 1)) and np.allclose(r[1:], 0)
    pairs = [(u, v) for u in range(5) for v in range(5) if u != v]
    K = oracle.Graph(5, [p[0] for p in pairs], [p[1] for p in pairs])
    assert np.allclose(K.bc(range(5)), 0)


def test_bc_parallel_edges_count_as_distinct_paths():
    # 0 =>(x2) 1 -> 3, 0 -> 2 -> 3 : sigma_03 = 3, through 1: 2, through 2: 1
    G = oracle.Graph(4, [0, 0, 1, 0, 2], [1, 1, 3, 2, 3])
    assert np.allclose(G.bc([0]), [0, 2 / 3, 1 / 3, 0])


# --------------------------------------------------------- partition, beta
def test_partition_golden_and_serpentine():
    g = GOLD["partition_degree_tie"]
    G = oracle.Graph(g["V"], g["src"], g["dst"])
    part, local = G.partition(1)
    assert list(local) == [g["order"].index(v) for v in range(3)], g["cite"]
    # degrees 5,4,3,2,1 on vertices 4,3,2,1,0 (ids reversed), P=2
    src = np.repeat(np.arange(5), [1, 2, 3, 4, 5]).astype(np.uint32)
    G = oracle.Graph(5, src, np.zeros(len(src), np.uint32))
    part, local = G.partition(2)
    # order 4,3,2,1,0 -> (p0,l0),(p1,l0),(p1,l1),(p0,l1),(p0,l2)
    exp = {4: (0, 0), 3: (1, 0), 2: (1, 1), 1: (0, 1), 0: (0, 2)}
    for v, (p, l) in exp.items():
        assert (part[v], local[v]) == (p, l)


def test_partition_balance_and_dense_local_ids():
    rng = np.random.default_rng(7)
    src, dst = random_multigraph(rng, 1000, 8000)
    G = oracle.Graph(1000, src, dst)
    for P in (1, 2, 3, 8):
        part, local = G.partition(P)
        for p in range(P):
            ids = np.sort(local[part == p])
            assert np.array_equal(ids, np.arange(len(ids)))
            assert abs(len(ids) - 1000 / P) <= 1


def test_partition_random_definition_and_invariants():
    """RAND partitioning (Fig. 4's random baseline): the partition depends
    only on the key draw, not on the edges; sizes equal the serpentine deal's;
    local ids are dense and follow out-degree desc, id asc inside each part.
    Checked against a hand-worked 6-vertex case and numpy lexsort."""
    import inputs

    # hand-worked: keys [5, 1, 5, 0, 9, 2] -> order 3,1,5,0,2,4 -> P=2 serpentine
    # parts 0,1,1,0,0,1 -> part[3]=0, part[1]=1, part[5]=1, part[0]=0, part[2]=0, part[4]=1
    src = np.array([0, 0, 0, 4, 4, 2], np.uint32)   # outdeg: 0:3, 4:2, 2:1, others 0
    dst = np.array([1, 2, 3, 5, 1, 0], np.uint32)
    G = oracle.Graph(6, src, dst)
    part, local = G.partition_random(2, np.array([5, 1, 5, 0, 9, 2], np.uint32))
    assert list(part) == [0, 1, 0, 0, 1, 1]
    # part 0 = {0 (deg 3), 2 (deg 1), 3 (deg 0)}; part 1 = {4 (deg 2), 1, 5 (deg 0)}
    assert list(local) == [0, 1, 1, 2, 0, 2]

    rng = np.random.default_rng(17)
    n = 3000
    src, dst = random_multigraph(rng, n, 20000)
    keys = inputs.part_keys(n)
    G = oracle.Graph(n, src, dst)
    deg = G.out_degree()
    G2 = oracle.Graph(n, dst, src)                      # other edges, same keys
    for P in (1, 2, 3, 8):
        part, local = G.partition_random(P, keys)
        assert np.array_equal(G2.partition_random(P, keys)[0], part)
        pos = np.empty(n, np.int64)
        pos[np.lexsort((np.arange(n), keys))] = np.arange(n)
        r, j = pos // P, pos % P
        assert np.array_equal(part, np.where(r % 2 == 0, j, P - 1 - j))
        for p in range(P):
            members = np.flatnonzero(part == p)
            want = members[np.lexsort((members, -deg[members].astype(np.int64)))]
            assert np.array_equal(local[want], np.arange(len(members)))
        sizes = np.bincount(part, minlength=P)
        dpart, _ = G.partition(P)
        assert np.array_equal(sizes, np.bincount(dpart, minlength=P))


def test_beta_golden_and_invariants():
    g = GOLD["beta_two_edges_one_remote"]
    br, bd, slots = oracle.beta(g["V"], g["src"], g["dst"], g["part"], g["P"])
    assert (br, bd) == (g["beta_raw"], g["beta_reduced"]), g["cite"]
    assert slots[0, 1] == 1 and slots[1, 0] == 0
    rng = np.random.default_rng(8)
    src, dst = random_multigraph(rng, 500, 5000)
    br, bd, _ = oracle.beta(500, src, dst, np.zeros(500, np.uint32), 1)
    assert br == 0 and bd == 0                             # single partition
    part = rng.integers(0, 2, 500).astype(np.uint32)
    br, bd, slots = oracle.beta(500, src, dst, part, 2)
    assert 0 <= bd <= br <= 1
    # duplicating every edge leaves beta_reduced * E invariant
    br2, bd2, slots2 = oracle.beta(500, np.r_[src, src], np.r_[dst, dst], part, 2)
    assert np.array_equal(slots, slots2) and np.isclose(br2, br)
    # brute force distinct pairs
    cross = part[src] != part[dst]
    pairs = {(int(part[s]), int(d)) for s, d in zip(src[cross], dst[cross])}
    assert np.isclose(bd * len(src), len(pairs))


# ----------------------------------------------- streaming (full-size) certificates
def test_streaming_certificates_match_in_memory_ones():
    rng = np.random.default_rng(9)
    n = 3000
    src, dst = random_multigraph(rng, n, 20000)
    w = rng.integers(1, 64, len(src)).astype(np.uint32)
    G = oracle.Graph(n, src, dst, w)
    for s in (0, 7):
        for weighted, truth in ((False, G.bfs(s)), (True, G.sssp(s))):
            cands = [truth]
            reached = np.where((truth != INF32) & (np.arange(n) != s))[0]
            for v in reached[:5]:
                for delta in (-1, 1):
                    bad = truth.copy(); bad[v] = int(truth[v]) + delta
                    cands.append(bad)
                bad = truth.copy(); bad[v] = INF32
                cands.append(bad)
            for k, vals in enumerate(cands):
                cert = oracle.StreamingCertificate(n, s, vals, weighted)
                for a in range(0, len(src), 4096):            # chunked feed
                    cert.feed(src[a:a + 4096], dst[a:a + 4096], w[a:a + 4096])
                assert cert.holds() == (k == 0)
                assert cert.holds() == (G.sssp_certify(s, vals) if weighted else G.bfs_certify(s, vals))


def test_pr_sample_recurrence_matches_oracle():
    rng = np.random.default_rng(10)
    n = 2000
    src, dst = random_multigraph(rng, n, 15000)
    G = oracle.Graph(n, src, dst)
    r4, r5 = G.pagerank(4), G.pagerank(5)
    outdeg = np.zeros(n, np.uint32)
    oracle.outdeg_edges(n, src, outdeg)
    assert np.array_equal(outdeg, G.out_degree().astype(np.uint32))
    sample = rng.choice(n, 300, replace=False)
    mask = np.zeros((n + 63) // 64, np.uint64)
    slot = np.zeros(n, np.uint32)
    for i, v in enumerate(sample):
        mask[v >> 6] |= np.uint64(1) << np.uint64(v & 63)
        slot[v] = i
    acc = np.zeros(len(sample))
    oracle.pr_sample_edges(n, src, dst, mask, slot, r4.astype(np.float32), outdeg, acc)
    pred = 0.15 / n + 0.85 * acc
    assert np.allclose(pred, r5[sample], rtol=1e-6)


def test_bc_single_source_dependency_identity():
    # sum_v delta_s(v) = sum_{t reachable, t != s} (d(s,t) - 1): every shortest
    # s-t path has d(s,t)-1 interior vertices (used at full size, where Brandes
    # cannot run on the host)
    rng = np.random.default_rng(12)
    for trial in range(20):
        n = int(rng.integers(2, 400))
        src, dst = random_multigraph(rng, n, int(rng.integers(1, 6 * n)))
        G = oracle.Graph(n, src, dst)
        s = int(rng.integers(0, n))
        lv = G.bfs(s).astype(np.int64)
        reached = (lv != INF32) & (np.arange(n) != s)
        assert np.isclose(G.bc([s]).sum(), (lv[reached] - 1).sum(), rtol=1e-12, atol=1e-9)


# ------------------------------------------------------------ connected components
def undirected_closure_labels(n, src, dst):
    """Brute force: boolean reachability closure of the symmetrised adjacency
    (repeated squaring), label = smallest reachable id (v reaches itself)."""
    A = np.eye(n, dtype=bool)
    for a, b in zip(src, dst):
        A[a, b] = A[b, a] = True
    for _ in range(max(1, int(np.ceil(np.log2(max(n, 2)))))):
        A = (A.astype(np.int64) @ A.astype(np.int64)) > 0
    return np.array([np.flatnonzero(A[v]).min() for v in range(n)], np.uint32)


def test_cc_golden():
    for key in ("cc_two_edges", "cc_path5"):
        g = GOLD[key]
        G = oracle.Graph(g["V"], g["src"], g["dst"])
        assert G.cc().tolist() == g["labels"], key


def test_cc_vs_brute_force_closure_and_direction_invariance():
    rng = np.random.default_rng(31)
    for _ in range(300):
        n = int(rng.integers(1, 9))
        src, dst = random_multigraph(rng, n, int(rng.integers(0, 2 * n)))
        want = undirected_closure_labels(n, src, dst)
        assert np.array_equal(oracle.Graph(n, src, dst).cc(), want)
        # weak components ignore edge direction
        assert np.array_equal(oracle.Graph(n, dst, src).cc(), want)


def test_cc_vs_scipy_weak_components():
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components

    rng = np.random.default_rng(32)
    for n, m in ((50, 30), (500, 400), (3000, 2500), (2000, 8000)):
        src, dst = random_multigraph(rng, n, m)
        A = coo_matrix((np.ones(len(src)), (src, dst)), shape=(n, n))
        k, comp = connected_components(A, directed=True, connection="weak")
        mins = np.full(k, n, np.int64)
        np.minimum.at(mins, comp, np.arange(n))
        lab = oracle.Graph(n, src, dst).cc()
        assert np.array_equal(lab, mins[comp].astype(np.uint32))
        assert len(np.unique(lab)) == k


def test_cc_streaming_equals_in_memory_and_invariants():
    rng = np.random.default_rng(33)
    n = 4000
    src, dst = random_multigraph(rng, n, 3500)
    want = oracle.Graph(n, src, dst).cc()
    S = oracle.StreamingCC(n)
    for i in range(0, len(src), 777):
        S.feed(src[i:i + 777], dst[i:i + 777])
    lab = S.labels()
    assert np.array_equal(lab, want)
    # label[v] <= v, labels are fixed points, and every edge joins equal labels
    assert (lab <= np.arange(n)).all() and np.array_equal(lab[lab], lab)
    assert np.array_equal(lab[src], lab[dst])
