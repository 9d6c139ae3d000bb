"""Host graphs and the text edge-list loader of the C ABI (tg_graph_*; SPEC
S:39-47 operation load_edge_list).  Host-only calls: no GPU needed.  The
expected values are the SPEC's examples (forced by the CSR definition) and the
error contract of include/tgraph.h."""
import numpy as np
import pytest

import paper_1312_3018_b200 as tg
from paper_1312_3018_b200.tgraph import TG_EINVAL, TG_EIO


def write(tmp_path, text, name="g.txt"):
    p = tmp_path / name
    p.write_text(text)
    return str(p)


def test_spec_path_example(tmp_path):
    # "0 1\n1 2", directed -> V=3, E=2
    g = tg.Graph.load_edge_list(write(tmp_path, "0 1\n1 2"))
    assert (g.V, g.E, g.weighted) == (3, 2, False)
    s, d, w = g.edges()
    assert s.tolist() == [0, 1] and d.tolist() == [1, 2] and w is None


def test_spec_empty_with_nodes_header(tmp_path):
    # empty file with "# nodes: 4" -> V=4, E=0
    g = tg.Graph.load_edge_list(write(tmp_path, "# nodes: 4\n"))
    assert (g.V, g.E) == (4, 0)


def test_spec_weighted_example(tmp_path):
    # "0 1 5\n0 2 7", weighted, directed -> weights [5, 7]
    g = tg.Graph.load_edge_list(write(tmp_path, "0 1 5\n0 2 7\n"), weighted=True)
    s, d, w = g.edges()
    assert g.weighted and s.tolist() == [0, 0] and d.tolist() == [1, 2] and w.tolist() == [5, 7]


def test_comments_blank_lines_crlf_and_duplicates(tmp_path):
    txt = "# a comment\n\n0 1\r\n  0   1  \n# nodes: 5\n3 3\n"
    g = tg.Graph.load_edge_list(write(tmp_path, txt))
    s, d, _ = g.edges()
    assert g.V == 5 and s.tolist() == [0, 0, 3] and d.tolist() == [1, 1, 3]  # multiset kept


def test_undirected_materialises_both_directions(tmp_path):
    g = tg.Graph.load_edge_list(write(tmp_path, "0 1 4\n1 2 9\n"), directed=False, weighted=True)
    s, d, w = g.edges()
    assert sorted(zip(s.tolist(), d.tolist(), w.tolist())) == [(0, 1, 4), (1, 0, 4), (1, 2, 9),
                                                              (2, 1, 9)]


@pytest.mark.parametrize("text,weighted,line,what", [
    ("0 1\n1 x\n", False, 2, "malformed"),
    ("0 1\n1\n", False, 2, "expected"),
    ("0 1 3\n1 2 -4\n", True, 2, "negative weight"),
    ("0 1\n1 2\n2\n", False, 3, "expected"),
    ("0 1 2 3\n", False, 1, "trailing"),
    ("0 1\n-1 2\n", False, 2, "negative vertex"),
    ("0 1\n1 2\n", True, 1, "missing weight"),
    ("# nodes: 2\n0 1\n1 2\n", False, 3, "declared"),
])
def test_errors_name_the_line(tmp_path, text, weighted, line, what):
    with pytest.raises(tg.TGraphError) as e:
        tg.Graph.load_edge_list(write(tmp_path, text), weighted=weighted)
    assert e.value.code == TG_EINVAL
    assert f"line {line}" in str(e.value) and what in str(e.value)


def test_missing_file_is_eio(tmp_path):
    with pytest.raises(tg.TGraphError) as e:
        tg.Graph.load_edge_list(str(tmp_path / "nope.txt"))
    assert e.value.code == TG_EIO


def test_empty_file_without_header_is_rejected(tmp_path):
    with pytest.raises(tg.TGraphError) as e:
        tg.Graph.load_edge_list(write(tmp_path, "# nothing\n"))
    assert e.value.code == TG_EINVAL


def test_from_edges_copies_and_validates():
    src = np.array([0, 2, 1], np.uint32)
    dst = np.array([1, 0, 2], np.uint32)
    g = tg.Graph.from_edges(3, src, dst)
    src[0] = 7  # the library copied its input
    s, d, _ = g.edges()
    assert s.tolist() == [0, 2, 1] and d.tolist() == [1, 0, 2] and not g.weighted
    with pytest.raises(tg.TGraphError) as e:
        tg.Graph.from_edges(2, np.array([0], np.uint32), np.array([2], np.uint32))
    assert e.value.code == TG_EINVAL


def test_engine_create_rejects_weighted_attr_on_unweighted_graph():
    g = tg.Graph.from_edges(2, np.array([0], np.uint32), np.array([1], np.uint32))
    with pytest.raises(tg.TGraphError) as e:
        tg.Engine.from_graph(g, weighted=True)
    assert e.value.code == TG_EINVAL


def test_rmat_slice_validates_before_the_device():
    with pytest.raises(tg.TGraphError) as e:
        tg.tg_rmat_edges(4, first=10, count=16 * 16)  # past the end of the stream
    assert e.value.code == TG_EINVAL
    with pytest.raises(tg.TGraphError) as e:
        tg.tg_rmat_edges(4, a=0.6, b=0.3, c=0.3, count=4)
    assert e.value.code == TG_EINVAL
