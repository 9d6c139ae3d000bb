"""Seeded input generator (inputs/tg_inputs.h).  Not an oracle: the generator
is shared input, so its "parity" is unpinned by construction; these
tests check the properties the paper fixes for the workload (PAPER.md:326,
Table 2: (A,B,C) = (0.57,0.19,0.19), degree 16, directed) and determinism."""
import numpy as np

import inputs


def test_edge_count_and_range():
    for s in (1, 5, 10):
        src, dst, _ = inputs.rmat_edges(s)
        assert len(src) == 16 << s  # E = 16 * 2^s (Table 2)
        assert src.max() < (1 << s) and dst.max() < (1 << s)


def test_degenerate_a1_all_edges_on_vertex0():
    # a=1 forces quadrant A at every level; scrambling off.
    src, dst, _ = inputs.rmat_edges(1, edge_factor=1, a=1.0, b=0.0, c=0.0, scramble=False)
    assert list(src) == [0, 0] and list(dst) == [0, 0]


def test_determinism_and_slices():
    a = inputs.rmat_edges(12, weights=True)
    b = inputs.rmat_edges(12, weights=True)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    s2, d2, w2 = inputs.rmat_edges(12, weights=True, first=1000, count=500)
    assert np.array_equal(s2, a[0][1000:1500]) and np.array_equal(w2, a[2][1000:1500])
    assert a[2].min() >= 1 and a[2].max() <= 63


def test_scramble_is_bijection():
    for s in (1, 2, 7, 12):
        vals = {inputs.scramble_one(x, s) for x in range(1 << s)}
        assert vals == set(range(1 << s))


def test_quadrant_bit_frequencies():
    # Without scrambling, each of the `scale` bits of (src, dst) is an
    # independent quadrant draw: P(src bit)=C+D=0.24, P(dst bit)=B+D=0.24,
    # P(both)=D=0.05 (Table 2 caption).  4-sigma binomial bounds.
    scale = 10
    src, dst, _ = inputs.rmat_edges(scale, scramble=False)
    n = len(src) * scale
    sb = sum(int(((src >> i) & 1).sum()) for i in range(scale))
    db = sum(int(((dst >> i) & 1).sum()) for i in range(scale))
    both = sum(int((((src & dst) >> i) & 1).sum()) for i in range(scale))
    for cnt, p in ((sb, 0.24), (db, 0.24), (both, 0.05)):
        assert abs(cnt - n * p) < 4 * np.sqrt(n * p * (1 - p))


def test_skew_max_degree():
    # Expected max out-degree ~ E * (A+B)^s = E * 0.76^s (the all-zero-bit row).
    scale = 14
    src, _, _ = inputs.rmat_edges(scale)
    maxdeg = np.bincount(src, minlength=1 << scale).max()
    expected = (16 << scale) * 0.76 ** scale
    assert 0.7 * expected < maxdeg < 1.3 * expected


def test_sources_have_out_edges():
    scale = 10
    src, _, _ = inputs.rmat_edges(scale)
    s = inputs.rmat_sources(scale, 64)
    deg = np.bincount(src, minlength=1 << scale)
    assert (deg[s.astype(np.int64)] >= 1).all()
    s2 = inputs.list_sources(src, 64)
    assert np.array_equal(s, s2)
