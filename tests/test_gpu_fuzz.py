"""GPU fuzz parity: many small seeded graphs of varied shape -- sparse / dense,
skewed hubs, chains, stars in and out, bipartite layers, duplicate edges,
self-loops, isolated vertices, wide weights -- each built over a random
partition count, strategy and transport, and every algorithm (BFS and SSSP
from several sources, PageRank, BC, CC) compared with the CPU oracle.  The
structured tests cover each feature on purpose; this sweep looks for the
combinations nobody wrote down.  Bars as in test_gpu_parity."""
import numpy as np
import pytest

import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tg():
    import paper_1312_3018_b200 as tg

    tg.lib()
    return tg


def _graph(rng, kind):
    """-> V, src, dst, w for one fuzz case."""
    V = int(rng.integers(2, 1500))
    if kind == "uniform":
        E = int(rng.integers(0, 8 * V))
        s, d = rng.integers(0, V, E), rng.integers(0, V, E)
    elif kind == "skewed":  # a few hubs take most endpoints
        E = int(rng.integers(V, 12 * V))
        hubs = rng.integers(0, V, max(1, V // 50))
        pick = rng.random(E) < 0.7
        s = np.where(pick, rng.choice(hubs, E), rng.integers(0, V, E))
        d = np.where(rng.random(E) < 0.5, rng.choice(hubs, E), rng.integers(0, V, E))
    elif kind == "chain":  # long paths: many supersteps
        perm = rng.permutation(V)
        s, d = perm[:-1], perm[1:]
        if rng.random() < 0.5:
            s, d = np.concatenate([s, d]), np.concatenate([d, s])
    elif kind == "stars":  # one out-star and one in-star of large degree
        c1, c2 = rng.integers(0, V, 2)
        s = np.concatenate([np.full(V, c1), rng.integers(0, V, V)])
        d = np.concatenate([rng.integers(0, V, V), np.full(V, c2)])
    else:  # "layers": bipartite layers, many equal-length shortest paths (BC sigma)
        L = int(rng.integers(2, 8))
        cut = np.sort(rng.choice(np.arange(1, V), size=min(L, V - 1), replace=False))
        layer = np.searchsorted(cut, np.arange(V), side="right")
        E = int(rng.integers(V, 6 * V))
        s = rng.integers(0, V, E)
        nxt = np.where(layer[s] < layer.max(), layer[s] + 1, layer[s])
        members = [np.where(layer == k)[0] for k in range(layer.max() + 1)]
        d = np.array([rng.choice(members[k]) if len(members[k]) else 0 for k in nxt], dtype=np.int64)
    s = np.asarray(s, np.int64) % V
    d = np.asarray(d, np.int64) % V
    if len(s) and rng.random() < 0.5:  # duplicates and self-loops
        k = int(rng.integers(1, max(2, len(s) // 5)))
        idx = rng.integers(0, len(s), k)
        s = np.concatenate([s, s[idx], idx % V])
        d = np.concatenate([d, d[idx], idx % V])
    wmax = int(rng.choice([1, 63, 255, 1 << 20]))
    w = rng.integers(1, wmax + 1, len(s))
    return V, s.astype(np.uint32), d.astype(np.uint32), w.astype(np.uint32)


def _max_sigma(V, s, d, source):
    """Largest exact shortest-path count (edge sequences, parallel edges
    distinct) from `source`, in Python integers."""
    adj = [[] for _ in range(V)]
    for a, b in zip(s.tolist(), d.tolist()):
        adj[a].append(b)
    lvl = [-1] * V
    sig = [0] * V
    lvl[source], sig[source] = 0, 1
    frontier = [source]
    while frontier:
        nxt = []
        for u in frontier:
            for v in adj[u]:
                if lvl[v] < 0:
                    lvl[v] = lvl[u] + 1
                    nxt.append(v)
                if lvl[v] == lvl[u] + 1:
                    sig[v] += sig[u]
        frontier = nxt
    return max(sig)


@pytest.mark.parametrize("seed", range(60))
def test_fuzz_all_algorithms(tg, seed):
    rng = np.random.default_rng(1000 + seed)
    kind = ["uniform", "skewed", "chain", "stars", "layers"][seed % 5]
    V, s, d, w = _graph(rng, kind)
    P = int(rng.choice([1, 2, 3, 5]))
    strategy = int(rng.choice([tg.TG_PART_DEGREE, tg.TG_PART_RANDOM]))
    G = oracle.Graph(V, s, d, w)
    eng = tg.Engine.from_edges(V, s, d, w, partitions=P, strategy=strategy)
    if P > 1 and rng.random() < 0.5:
        eng.set_exchange(tg.TG_EXCHANGE_COPY)
    if P > 1 and rng.random() < 0.5:
        eng.set_pagerank_comm(tg.TG_PR_PULL)
    deg = G.out_degree()
    cand = np.where(deg > 0)[0]
    srcs = [int(x) for x in rng.choice(cand, size=min(3, len(cand)), replace=False)] if len(cand) else []
    srcs.append(int(rng.integers(0, V)))  # possibly isolated / sink source
    for x in srcs:
        assert np.array_equal(eng.bfs(x)[0], G.bfs(x)), (kind, P, "bfs", x)
        assert np.array_equal(eng.sssp(x)[0], G.sssp(x)), (kind, P, "sssp", x)
    T = int(rng.integers(1, 8))
    ref = G.pagerank(T)
    got = eng.pagerank(T)[0].astype(np.float64)
    assert (np.abs(got - ref) / ref).max() <= 1e-5, (kind, P, "pagerank")
    bs = srcs[:2]
    if max(_max_sigma(V, s, d, x) for x in bs) >= 1 << 53:
        # reading A11: a path count that fp64 cannot hold exactly is an error
        with pytest.raises(tg.TGraphError) as e:
            eng.bc(np.asarray(bs, np.uint64))
        assert e.value.code == tg.tgraph.TG_EINTERNAL
    else:
        bref = G.bc(bs)
        bgot = eng.bc(np.asarray(bs, np.uint64))[0]
        scale = max(1.0, float(np.abs(bref).max()))
        assert (np.abs(bgot - bref) <= 1e-4 * np.abs(bref) + 1e-12 * scale).all(), (kind, P, "bc")
    assert np.array_equal(eng.cc()[0], G.cc()), (kind, P, "cc")
    eng.close()
