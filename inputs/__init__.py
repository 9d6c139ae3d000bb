"""ctypes binding of the seeded input generators (inputs/tg_inputs.c).

Shared by tests/, the oracle harness and bench.py.  Holds none of the method's
arithmetic: only the counter-based RMAT edge stream, SSSP weights and run
sources defined in tg_inputs.h.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

# Paper workload parameters: PAPER.md:326 (Table 2 caption) and DESIGN.md 8(d).
RMAT_A, RMAT_B, RMAT_C = 0.57, 0.19, 0.19
EDGE_FACTOR = 16
GRAPH_SEED, WEIGHT_SEED, SOURCE_SEED = 1, 2, 3
PART_SEED = 4  # TG_PART_RANDOM draw (tg_attr.part_seed default of the binding)


def lib():
    global _LIB
    if _LIB is None:
        import sys

        sys.path.insert(0, os.path.join(os.path.dirname(_HERE), "scripts"))
        from build import build_inputs  # type: ignore

        path = build_inputs()
        L = C.CDLL(path)
        u64, i32, dbl, p32, p64 = C.c_uint64, C.c_int, C.c_double, C.c_void_p, C.c_void_p
        L.tgin_rmat_edges.argtypes = [i32, i32, dbl, dbl, dbl, u64, i32, u64, u64, u64, p32, p32, p32]
        L.tgin_rmat_edges.restype = i32
        L.tgin_weights.argtypes = [u64, u64, u64, p32]
        L.tgin_weights.restype = i32
        L.tgin_rmat_sources.argtypes = [i32, i32, dbl, dbl, dbl, u64, i32, u64, u64, p64]
        L.tgin_rmat_sources.restype = i32
        L.tgin_list_sources.argtypes = [u64, p32, u64, u64, p64]
        L.tgin_list_sources.restype = i32
        L.tgin_scramble_one.argtypes = [C.c_uint32, i32, u64]
        L.tgin_scramble_one.restype = C.c_uint32
        L.tgin_part_keys.argtypes = [u64, u64, p32]
        L.tgin_part_keys.restype = i32
        _LIB = L
    return _LIB


def _ptr(a: np.ndarray | None):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


def rmat_edges(scale: int, edge_factor: int = EDGE_FACTOR, a: float = RMAT_A, b: float = RMAT_B,
               c: float = RMAT_C, seed: int = GRAPH_SEED, scramble: bool = True,
               weights: bool = False, wseed: int = WEIGHT_SEED, first: int = 0,
               count: int | None = None):
    """Edges [first, first+count) of the RMAT stream -> (src u32, dst u32, w u32 | None)."""
    E = edge_factor << scale
    if count is None:
        count = E - first
    src = np.empty(count, np.uint32)
    dst = np.empty(count, np.uint32)
    w = np.empty(count, np.uint32) if weights else None
    rc = lib().tgin_rmat_edges(scale, edge_factor, a, b, c, seed, int(scramble), wseed, first,
                               count, _ptr(src), _ptr(dst), _ptr(w))
    if rc != 0:
        raise ValueError(f"tgin_rmat_edges: invalid parameters (rc={rc})")
    return src, dst, w


def weights_for(count: int, wseed: int = WEIGHT_SEED, first: int = 0) -> np.ndarray:
    w = np.empty(count, np.uint32)
    if lib().tgin_weights(wseed, first, count, _ptr(w)) != 0:
        raise ValueError("tgin_weights")
    return w


def rmat_sources(scale: int, k: int, edge_factor: int = EDGE_FACTOR, a: float = RMAT_A,
                 b: float = RMAT_B, c: float = RMAT_C, seed: int = GRAPH_SEED,
                 scramble: bool = True, sseed: int = SOURCE_SEED) -> np.ndarray:
    out = np.empty(k, np.uint64)
    if lib().tgin_rmat_sources(scale, edge_factor, a, b, c, seed, int(scramble), sseed, k,
                               _ptr(out)) != 0:
        raise ValueError("tgin_rmat_sources")
    return out


def list_sources(src: np.ndarray, k: int, sseed: int = SOURCE_SEED) -> np.ndarray:
    src = np.ascontiguousarray(src, np.uint32)
    out = np.empty(k, np.uint64)
    if lib().tgin_list_sources(len(src), _ptr(src), sseed, k, _ptr(out)) != 0:
        raise ValueError("tgin_list_sources")
    return out


def scramble_one(x: int, scale: int, seed: int = GRAPH_SEED) -> int:
    return int(lib().tgin_scramble_one(x, scale, seed))


def part_keys(V: int, pseed: int = PART_SEED) -> np.ndarray:
    """Sort keys of the TG_PART_RANDOM draw (tgin_part_key) for vertices [0, V)."""
    out = np.empty(V, np.uint32)
    if lib().tgin_part_keys(pseed, V, _ptr(out)) != 0:
        raise ValueError("tgin_part_keys")
    return out
