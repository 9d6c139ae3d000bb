"""ctypes binding of the CPU oracle (oracle/oracle.c).

TEST INFRASTRUCTURE ONLY: imported by tests/, __graft_entry__.smoke() and
bench.py's cpu_baseline / --impl reference legs, never by the product package
paper_1312_3018_b200/.  See oracle.h for the definitions each function writes
out and DESIGN.md "Oracle pins" for what pins them.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None
INF32 = 0xFFFFFFFF


def lib():
    global _LIB
    if _LIB is None:
        import sys

        sys.path.insert(0, os.path.join(os.path.dirname(_HERE), "scripts"))
        from build import build_oracle  # type: ignore

        L = C.CDLL(build_oracle())
        u64, i32, dbl, p = C.c_uint64, C.c_int, C.c_double, C.c_void_p
        L.oracle_csr.argtypes = [u64, u64, p, p, p, p, p, p]
        L.oracle_bfs.argtypes = [u64, p, p, u64, p]
        L.oracle_sssp.argtypes = [u64, p, p, p, u64, p]
        L.oracle_pagerank.argtypes = [u64, p, p, i32, dbl, p]
        L.oracle_bc.argtypes = [u64, p, p, p, i32, p]
        L.oracle_partition.argtypes = [u64, p, i32, p, p]
        L.oracle_partition_random.argtypes = [u64, p, i32, p, p, p]
        L.oracle_beta.argtypes = [u64, u64, p, p, p, i32, p, p, p]
        L.oracle_bfs_certify.argtypes = [u64, p, p, u64, p, p]
        L.oracle_sssp_certify.argtypes = [u64, p, p, p, u64, p, p]
        L.oracle_outdeg_edges.argtypes = [u64, u64, p, p]
        L.oracle_bfs_cert_edges.argtypes = [u64, p, u64, p, p, p, p]
        L.oracle_sssp_cert_edges.argtypes = [u64, p, u64, p, p, p, p, p]
        L.oracle_cert_finish.argtypes = [u64, u64, p, p, p]
        L.oracle_pr_sample_edges.argtypes = [u64, u64, p, p, p, p, p, p, p]
        L.oracle_cc.argtypes = [u64, p, p, p]
        L.oracle_cc_edges.argtypes = [u64, p, u64, p, p]
        L.oracle_cc_finish.argtypes = [u64, p, p]
        for f in ("oracle_csr", "oracle_bfs", "oracle_sssp", "oracle_pagerank", "oracle_bc",
                  "oracle_partition", "oracle_partition_random", "oracle_beta", "oracle_bfs_certify",
                  "oracle_sssp_certify", "oracle_outdeg_edges", "oracle_bfs_cert_edges",
                  "oracle_sssp_cert_edges", "oracle_cert_finish", "oracle_pr_sample_edges",
                  "oracle_cc", "oracle_cc_edges", "oracle_cc_finish"):
            getattr(L, f).restype = i32
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def _check(rc: int, name: str) -> None:
    if rc != 0:
        raise RuntimeError(f"{name} failed with code {rc}")


class Graph:
    """Oracle-side CSR (its own; never the CUDA path's)."""

    def __init__(self, V: int, src, dst, w=None):
        self.V = int(V)
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        self.E = len(src)
        self.row_off = np.empty(self.V + 1, np.uint64)
        self.col = np.empty(max(self.E, 1), np.uint32)
        self.w = None
        wv = None
        if w is not None:
            wv = np.ascontiguousarray(w, np.uint32)
            self.w = np.empty(max(self.E, 1), np.uint32)
        _check(lib().oracle_csr(self.V, self.E, _p(src), _p(dst), _p(wv), _p(self.row_off),
                                _p(self.col), _p(self.w)), "oracle_csr")

    def out_degree(self) -> np.ndarray:
        return np.diff(self.row_off)

    def bfs(self, s: int) -> np.ndarray:
        lv = np.empty(self.V, np.uint32)
        _check(lib().oracle_bfs(self.V, _p(self.row_off), _p(self.col), s, _p(lv)), "oracle_bfs")
        return lv

    def sssp(self, s: int) -> np.ndarray:
        d = np.empty(self.V, np.uint32)
        _check(lib().oracle_sssp(self.V, _p(self.row_off), _p(self.col), _p(self.w), s, _p(d)),
               "oracle_sssp")
        return d

    def pagerank(self, T: int = 5, d: float = 0.85) -> np.ndarray:
        r = np.empty(self.V, np.float64)
        _check(lib().oracle_pagerank(self.V, _p(self.row_off), _p(self.col), T, d, _p(r)),
               "oracle_pagerank")
        return r

    def bc(self, sources) -> np.ndarray:
        s = np.ascontiguousarray(sources, np.uint64)
        out = np.empty(self.V, np.float64)
        _check(lib().oracle_bc(self.V, _p(self.row_off), _p(self.col), _p(s), len(s), _p(out)),
               "oracle_bc")
        return out

    def cc(self) -> np.ndarray:
        """Weakly connected components: label = smallest id of the component."""
        out = np.empty(self.V, np.uint32)
        _check(lib().oracle_cc(self.V, _p(self.row_off), _p(self.col), _p(out)), "oracle_cc")
        return out

    def partition(self, P: int):
        part = np.empty(self.V, np.uint32)
        local = np.empty(self.V, np.uint32)
        _check(lib().oracle_partition(self.V, _p(self.row_off), P, _p(part), _p(local)),
               "oracle_partition")
        return part, local

    def partition_random(self, P: int, key):
        """RAND partitioning (oracle_partition_random); key = inputs.part_keys(V, seed)."""
        key = np.ascontiguousarray(key, np.uint32)
        part = np.empty(self.V, np.uint32)
        local = np.empty(self.V, np.uint32)
        _check(lib().oracle_partition_random(self.V, _p(self.row_off), P, _p(key), _p(part),
                                             _p(local)), "oracle_partition_random")
        return part, local

    def bfs_certify(self, s: int, level) -> bool:
        lv = np.ascontiguousarray(level, np.uint32)
        bad = np.zeros(1, np.uint64)
        return lib().oracle_bfs_certify(self.V, _p(self.row_off), _p(self.col), s, _p(lv),
                                        _p(bad)) == 0

    def sssp_certify(self, s: int, dist) -> bool:
        dv = np.ascontiguousarray(dist, np.uint32)
        bad = np.zeros(1, np.uint64)
        return lib().oracle_sssp_certify(self.V, _p(self.row_off), _p(self.col), _p(self.w), s,
                                         _p(dv), _p(bad)) == 0


def beta(V: int, src, dst, part, P: int):
    """(beta_raw, beta_reduced, slots[P,P]) per oracle_beta."""
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    part = np.ascontiguousarray(part, np.uint32)
    br, bd = np.zeros(1, np.float64), np.zeros(1, np.float64)
    slots = np.zeros((P, P), np.uint64)
    _check(lib().oracle_beta(V, len(src), _p(src), _p(dst), _p(part), P, _p(br), _p(bd),
                             _p(slots)), "oracle_beta")
    return float(br[0]), float(bd[0]), slots


class StreamingCertificate:
    """BFS / SSSP certificate over an edge stream fed in chunks (oracle.h
    streaming section): exact for graphs too large for an in-memory CSR."""

    def __init__(self, V: int, source: int, values, weighted: bool):
        self.V, self.s, self.weighted = int(V), int(source), weighted
        self.val = np.ascontiguousarray(values, np.uint32)
        self.tight = np.zeros((self.V + 63) // 64, np.uint64)
        self.bad = np.zeros(1, np.uint64)

    def feed(self, src, dst, w=None) -> None:
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        if self.weighted:
            w = np.ascontiguousarray(w, np.uint32)
            rc = lib().oracle_sssp_cert_edges(self.V, _p(self.val), len(src), _p(src), _p(dst),
                                              _p(w), _p(self.tight), _p(self.bad))
        else:
            rc = lib().oracle_bfs_cert_edges(self.V, _p(self.val), len(src), _p(src), _p(dst),
                                             _p(self.tight), _p(self.bad))
        _check(rc, "streaming certificate")

    def holds(self) -> bool:
        if int(self.bad[0]):
            return False
        b = np.zeros(1, np.uint64)
        return lib().oracle_cert_finish(self.V, self.s, _p(self.val), _p(self.tight), _p(b)) == 0


class StreamingCC:
    """Union-find connected components over an edge stream fed in chunks."""

    def __init__(self, V: int):
        self.V = int(V)
        self.parent = np.arange(self.V, dtype=np.uint32)

    def feed(self, src, dst) -> None:
        src = np.ascontiguousarray(src, np.uint32)
        dst = np.ascontiguousarray(dst, np.uint32)
        _check(lib().oracle_cc_edges(self.V, _p(self.parent), len(src), _p(src), _p(dst)),
               "oracle_cc_edges")

    def labels(self) -> np.ndarray:
        out = np.empty(self.V, np.uint32)
        _check(lib().oracle_cc_finish(self.V, _p(self.parent), _p(out)), "oracle_cc_finish")
        return out


def outdeg_edges(V: int, src, outdeg: np.ndarray) -> None:
    src = np.ascontiguousarray(src, np.uint32)
    _check(lib().oracle_outdeg_edges(V, len(src), _p(src), _p(outdeg)), "oracle_outdeg_edges")


def pr_sample_edges(V: int, src, dst, mask, slot, r_prev, outdeg, acc) -> None:
    src = np.ascontiguousarray(src, np.uint32)
    dst = np.ascontiguousarray(dst, np.uint32)
    _check(lib().oracle_pr_sample_edges(V, len(src), _p(src), _p(dst), _p(mask), _p(slot),
                                        _p(r_prev), _p(outdeg), _p(acc)), "oracle_pr_sample_edges")
