"""GPU parity for connected components (tg_cc): the CUDA
label propagation through the C ABI against the oracle's union-find, element by
element (labels are integers: bit-exact)."""
import json
import os

import numpy as np
import pytest

import inputs
import oracle

pytestmark = pytest.mark.gpu

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


@pytest.fixture(scope="module")
def tg():
    import paper_1312_3018_b200 as tg

    tg.lib()
    return tg


def run(tg, V, src, dst, P=1):
    eng = tg.Engine.from_edges(V, np.asarray(src, np.uint32), np.asarray(dst, np.uint32),
                               partitions=P)
    return eng.cc()


@pytest.mark.parametrize("P", [1, 2, 3])
def test_cc_golden(tg, P):
    for key in ("cc_two_edges", "cc_path5"):
        g = GOLD[key]
        lab, st = run(tg, g["V"], g["src"], g["dst"], P=P)
        assert lab.tolist() == g["labels"], g["cite"]
        if "max_supersteps" in g:
            # the path converges within 5 supersteps (the extra
            # one is the superstep whose vote finds no change)
            assert st.supersteps <= g["max_supersteps"] + 1


@pytest.mark.parametrize("P", [1, 2, 4])
def test_cc_random_multigraphs(tg, P):
    rng = np.random.default_rng(40 + P)
    for n, m in ((1, 0), (2, 1), (7, 3), (64, 40), (500, 300), (3000, 2000), (4000, 12000)):
        src = rng.integers(0, n, m)
        dst = rng.integers(0, n, m)
        if P > n:
            continue
        want = oracle.Graph(n, src, dst).cc()
        got, _ = run(tg, n, src, dst, P=P)
        assert np.array_equal(got, want), (n, m)


def test_cc_long_path_both_orientations(tg):
    # labels must flow against edge direction too (weak components): a path
    # whose edges all point towards vertex 0 only converges through the in-CSR
    n = 3000
    perm = np.random.default_rng(5).permutation(n)
    src, dst = perm[1:], perm[:-1]            # edges point "down" the path
    for P in (1, 2, 5):
        for s, d in ((src, dst), (dst, src)):
            got, st = run(tg, n, s, d, P=P)
            assert (got == 0).all()
            assert st.traversed_edges == n - 1


@pytest.mark.parametrize("P", [1, 3, 8])
def test_cc_rmat12(tg, P):
    scale = 12
    src, dst, _ = inputs.rmat_edges(scale)
    want = oracle.Graph(1 << scale, src, dst).cc()
    eng = tg.Engine.rmat(scale, partitions=P)      # device-side generation
    assert np.array_equal(eng.cc()[0], want)
    eng_up = tg.Engine.from_edges(1 << scale, src, dst, partitions=P)
    assert np.array_equal(eng_up.cc()[0], want)


def test_cc_uniform_and_sparse_many_components(tg):
    # edge factor 1 uniform graph: many small components + isolated vertices
    scale = 14
    src, dst, _ = inputs.rmat_edges(scale, edge_factor=1, a=0.25, b=0.25, c=0.25)
    want = oracle.Graph(1 << scale, src, dst).cc()
    assert len(np.unique(want)) > 1000
    for P in (1, 4):
        eng = tg.Engine.rmat(scale, edge_factor=1, a=0.25, b=0.25, c=0.25, partitions=P)
        assert np.array_equal(eng.cc()[0], want)


def test_cc_device_output_and_errors(tg):
    import torch

    scale = 10
    src, dst, _ = inputs.rmat_edges(scale)
    want = oracle.Graph(1 << scale, src, dst).cc()
    eng = tg.Engine.rmat(scale)
    out = torch.empty(1 << scale, dtype=torch.int32, device="cuda")
    eng.cc(out=out)
    assert np.array_equal(out.cpu().numpy().view(np.uint32), want)
    eng2 = tg.Engine.from_edges(1 << scale, src, dst, in_csr=False)
    with pytest.raises(tg.TGraphError) as e:
        eng2.cc()                                   # needs the in-CSR
    assert e.value.code == 2


def test_cc_c2_rmat22(tg):
    scale = 22
    src, dst, _ = inputs.rmat_edges(scale)
    want = oracle.Graph(1 << scale, src, dst).cc()
    del src, dst
    eng = tg.Engine.rmat(scale, weighted=False)
    got, st = eng.cc()
    assert np.array_equal(got, want)
    assert st.traversed_edges == 16 << scale
