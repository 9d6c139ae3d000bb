"""ctypes binding of libtgraph.so -- same names as include/tgraph.h.

Arrays: numpy arrays are host memory (TG_MEM_HOST); torch CUDA tensors are
device memory (TG_MEM_DEVICE, passed by data_ptr()).  Nothing here computes:
each function marshals arguments, calls the C ABI and raises TGraphError on a
non-zero status with tg_last_error().
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libtgraph.so")

TG_OK, TG_EINVAL, TG_ECAPACITY, TG_EIO, TG_EINTERNAL, TG_ECUDA, TG_ENCCL = 0, 2, 3, 4, 5, 6, 7
TG_MEM_HOST, TG_MEM_DEVICE = 0, 1
TG_INF32 = 0xFFFFFFFF


class TGraphError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[tg status {code}] {msg}")
        self.code = code


ALLGATHER_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_void_p, C.c_uint64)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_uint64), C.c_int, C.c_int)


class tg_comm(C.Structure):
    _fields_ = [("ctx", C.c_void_p), ("allgather", ALLGATHER_FN), ("allreduce_u64", ALLREDUCE_FN)]


class tg_attr(C.Structure):
    _fields_ = [("num_partitions", C.c_int), ("device", C.c_int), ("weighted", C.c_int),
                ("build_in_csr", C.c_int), ("rank", C.c_int), ("world", C.c_int),
                ("comm", C.POINTER(tg_comm)), ("strategy", C.c_int), ("part_seed", C.c_int)]


_U64_MAX = (1 << 64) - 1
_I64_MAX = (1 << 63) - 1


class TorchComm:
    """tg_comm backed by torch.distributed (gloo or nccl): the library's host
    collectives for metadata, the per-superstep vote and barriers.  Boundary
    messages never go through here (they are peer-memory copies)."""

    def __init__(self, group=None):
        import torch
        import torch.distributed as dist

        self.group = group
        self.world = dist.get_world_size(group)
        self.device = "cuda" if dist.get_backend(group) == "nccl" else "cpu"

        def allgather(ctx, send, recv, nbytes):
            try:
                src = np.frombuffer((C.c_ubyte * nbytes).from_address(send), np.uint8).copy()
                t = torch.from_numpy(src).to(self.device)
                outs = [torch.empty_like(t) for _ in range(self.world)]
                dist.all_gather(outs, t, group=group)
                res = torch.cat(outs).cpu().numpy()
                C.memmove(recv, res.ctypes.data, self.world * nbytes)
                return 0
            except Exception:  # noqa: BLE001 -- reported to C as a status
                return 1

        def allreduce(ctx, data, n, op):
            try:
                vals = [int(data[i]) for i in range(n)]
                if op == 1:  # min: keep the all-ones sentinel representable in int64
                    vals = [_I64_MAX if v == _U64_MAX else v for v in vals]
                else:        # sum modulo 2^64 via two's complement int64
                    vals = [v - (1 << 64) if v > _I64_MAX else v for v in vals]
                t = torch.tensor(vals, dtype=torch.int64, device=self.device)
                dist.all_reduce(t, op=dist.ReduceOp.MIN if op == 1 else dist.ReduceOp.SUM,
                                group=group)
                for i, v in enumerate(t.cpu().tolist()):
                    data[i] = _U64_MAX if (op == 1 and v == _I64_MAX) else v % (1 << 64)
                return 0
            except Exception:  # noqa: BLE001
                return 1

        self._ag = ALLGATHER_FN(allgather)
        self._ar = ALLREDUCE_FN(allreduce)
        self.struct = tg_comm(None, self._ag, self._ar)


class tg_info(C.Structure):
    _fields_ = [("V", C.c_uint64), ("E", C.c_uint64), ("num_partitions", C.c_int),
                ("weighted", C.c_int), ("has_in_csr", C.c_int), ("device_bytes", C.c_uint64),
                ("build_ms", C.c_uint64), ("device", C.c_int), ("strategy", C.c_int),
                ("exchange", C.c_int), ("pr_comm", C.c_int), ("peer_probe", C.c_int)]


class tg_part_info(C.Structure):
    _fields_ = [("Vp", C.c_uint64), ("Ep", C.c_uint64), ("Ep_local", C.c_uint64),
                ("outbox_slots", C.c_uint64), ("inbox_slots", C.c_uint64)]


class tg_stats(C.Structure):
    _fields_ = [("device_ms", C.c_double), ("supersteps", C.c_uint64),
                ("traversed_edges", C.c_uint64), ("algorithmic_bytes", C.c_uint64),
                ("comm_bytes", C.c_uint64), ("launches", C.c_uint64),
                ("relaxations", C.c_uint64), ("compute_ms", C.c_double),
                ("exchange_ms", C.c_double), ("vote_ms", C.c_double)]


class tg_kernel_stat(C.Structure):
    _fields_ = [("launches", C.c_uint64), ("ms", C.c_double), ("algorithmic_bytes", C.c_double)]


TG_K_COUNT = 9


@dataclass
class Stats:
    device_ms: float
    supersteps: int
    traversed_edges: int
    algorithmic_bytes: int
    comm_bytes: int
    launches: int
    relaxations: int = 0
    compute_ms: float = 0.0
    exchange_ms: float = 0.0
    vote_ms: float = 0.0

    @staticmethod
    def of(s: tg_stats) -> "Stats":
        return Stats(*(getattr(s, f) for f, _ in tg_stats._fields_))


_LIB = None


def lib():
    """Load libtgraph.so (built in-tree by __graft_entry__.build())."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; "
                              "g.build()'` (no CPU fallback exists)")
        L = C.CDLL(LIB_PATH)
        p, u64, i32, dbl = C.c_void_p, C.c_uint64, C.c_int, C.c_double
        L.tg_version.restype = C.c_char_p
        L.tg_last_error.restype = C.c_char_p
        L.tg_engine_create_edges.argtypes = [u64, u64, p, p, p, i32, C.POINTER(tg_attr), C.POINTER(p)]
        L.tg_engine_create_rmat.argtypes = [i32, i32, dbl, dbl, dbl, u64, i32, u64,
                                            C.POINTER(tg_attr), C.POINTER(p)]
        L.tg_engine_free.argtypes = [p]
        L.tg_engine_free.restype = None
        L.tg_engine_info.argtypes = [p, C.POINTER(tg_info)]
        L.tg_engine_partition_info.argtypes = [p, i32, C.POINTER(tg_part_info), p]
        L.tg_bfs.argtypes = [p, u64, p, i32, C.POINTER(tg_stats)]
        L.tg_sssp.argtypes = [p, u64, p, i32, C.POINTER(tg_stats)]
        L.tg_pagerank.argtypes = [p, i32, dbl, p, i32, C.POINTER(tg_stats)]
        L.tg_bc.argtypes = [p, p, i32, p, i32, C.POINTER(tg_stats)]
        L.tg_cc.argtypes = [p, p, i32, C.POINTER(tg_stats)]
        L.tg_partition_size.argtypes = [u64, i32, i32, C.POINTER(C.c_uint64)]
        L.tg_partition_size.restype = i32
        L.tg_engine_set_profiling.argtypes = [p, i32]
        L.tg_engine_set_exchange.argtypes = [p, i32]
        L.tg_engine_set_pagerank_comm.argtypes = [p, i32]
        L.tg_device_die_map.argtypes = [i32, p, i32, C.POINTER(i32), C.POINTER(i32)]
        L.tg_engine_last_ticket.argtypes = [p, C.POINTER(C.c_uint64)]
        L.tg_engine_wait_ticket.argtypes = [p, u64]
        L.tg_engine_kernel_stat.argtypes = [p, i32, C.POINTER(tg_kernel_stat)]
        L.tg_kernel_name.argtypes = [i32]
        L.tg_kernel_name.restype = C.c_char_p
        L.tg_graph_from_edges.argtypes = [u64, u64, p, p, p, C.POINTER(p)]
        L.tg_graph_load_edge_list.argtypes = [C.c_char_p, i32, i32, C.POINTER(p)]
        L.tg_graph_info.argtypes = [p, C.POINTER(C.c_uint64), C.POINTER(C.c_uint64), C.POINTER(i32)]
        L.tg_graph_edges.argtypes = [p, p, p, p]
        L.tg_graph_free.argtypes = [p]
        L.tg_graph_free.restype = None
        L.tg_engine_create.argtypes = [p, C.POINTER(tg_attr), C.POINTER(p)]
        L.tg_rmat_edges.argtypes = [i32, i32, dbl, dbl, dbl, u64, i32, u64, u64, u64, p, p, p, i32]
        L.tg_engine_set_async_collect.argtypes = [p, i32]
        L.tg_engine_sync.argtypes = [p]
        L.tg_hostcomm_create.argtypes = [C.POINTER(tg_comm), i32, i32, C.POINTER(p)]
        L.tg_hostcomm_allreduce_u64.argtypes = [p, p, i32, p]
        L.tg_hostcomm_free.argtypes = [p]
        L.tg_hostcomm_free.restype = None
        for f in ("tg_engine_set_async_collect", "tg_engine_sync", "tg_hostcomm_create", "tg_hostcomm_allreduce_u64", "tg_engine_create_edges", "tg_engine_create_rmat", "tg_engine_info",
                  "tg_engine_partition_info", "tg_bfs", "tg_sssp", "tg_pagerank", "tg_bc",
                  "tg_cc", "tg_engine_set_profiling", "tg_engine_set_exchange", "tg_engine_set_pagerank_comm", "tg_device_die_map", "tg_engine_last_ticket", "tg_engine_wait_ticket", "tg_engine_kernel_stat", "tg_graph_from_edges",
                  "tg_graph_load_edge_list", "tg_graph_info", "tg_graph_edges", "tg_engine_create",
                  "tg_rmat_edges"):
            getattr(L, f).restype = i32
        _LIB = L
    return _LIB


def _check(rc: int) -> None:
    if rc != TG_OK:
        raise TGraphError(rc, lib().tg_last_error().decode())


def _arr(a, dtype):
    """-> (pointer, mem kind, keepalive)."""
    if a is None:
        return None, TG_MEM_HOST, None
    if hasattr(a, "data_ptr") and getattr(a, "is_cuda", False):
        return C.c_void_p(a.data_ptr()), TG_MEM_DEVICE, a
    arr = np.ascontiguousarray(a, dtype)
    return arr.ctypes.data_as(C.c_void_p), TG_MEM_HOST, arr


TG_PART_DEGREE, TG_PART_RANDOM = 0, 1


def _attr(partitions, device, weighted, in_csr, rank=0, world=1, comm=None, strategy=TG_PART_DEGREE,
          part_seed=4) -> tg_attr:
    at = tg_attr()
    at.num_partitions, at.device, at.weighted, at.build_in_csr = partitions, device, int(weighted), int(in_csr)
    at.rank, at.world = rank, world
    at.strategy, at.part_seed = int(strategy), int(part_seed)
    if comm is not None:
        at.comm = C.pointer(comm.struct)
    return at


def tg_engine_create_edges(V, src, dst, w=None, partitions=1, device=0, weighted=None, in_csr=True,
                           rank=0, world=1, comm=None, strategy=TG_PART_DEGREE, part_seed=4):
    ps, ms, k1 = _arr(src, np.uint32)
    pd, md, k2 = _arr(dst, np.uint32)
    pw, mw, k3 = _arr(w, np.uint32)
    E = len(src)
    if E and ms != md:
        raise ValueError("src and dst must live in the same memory")
    if weighted is None:
        weighted = w is not None
    at = _attr(partitions, device, weighted, in_csr, rank, world, comm, strategy, part_seed)
    h = C.c_void_p()
    _check(lib().tg_engine_create_edges(V, E, ps, pd, pw, ms, C.byref(at), C.byref(h)))
    return h


def tg_engine_create_rmat(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, scramble=True,
                          wseed=2, partitions=1, device=0, weighted=True, in_csr=True, rank=0,
                          world=1, comm=None, strategy=TG_PART_DEGREE, part_seed=4):
    at = _attr(partitions, device, weighted, in_csr, rank, world, comm, strategy, part_seed)
    h = C.c_void_p()
    _check(lib().tg_engine_create_rmat(scale, edge_factor, a, b, c, seed, int(scramble), wseed,
                                       C.byref(at), C.byref(h)))
    return h


def tg_rmat_edges(scale, edge_factor=16, a=0.57, b=0.19, c=0.19, seed=1, scramble=True, wseed=2,
                  first=0, count=None, weights=False, out=None):
    """Slice [first, first+count) of the RMAT stream, generated on the current
    CUDA device -> (src, dst, w|None) numpy u32 (or into `out` = (src, dst, w)
    device tensors)."""
    E = edge_factor << scale
    count = E - first if count is None else count
    if out is None:
        src, dst = np.empty(count, np.uint32), np.empty(count, np.uint32)
        w = np.empty(count, np.uint32) if weights else None
    else:
        src, dst, w = out
    ps, ms, k1 = _arr(src, np.uint32)
    pd, md, k2 = _arr(dst, np.uint32)
    pw, mw, k3 = _arr(w, np.uint32)
    if ms != md or (w is not None and mw != ms):
        raise ValueError("src, dst and w must live in the same memory")
    _check(lib().tg_rmat_edges(scale, edge_factor, a, b, c, seed, int(scramble), wseed, first, count,
                               ps, pd, pw, ms))
    return src, dst, w


class Graph:
    """Library-owned host edge list (tg_graph): the load step."""

    def __init__(self, handle):
        self.h = handle
        V, E, wt = C.c_uint64(), C.c_uint64(), C.c_int()
        _check(lib().tg_graph_info(handle, C.byref(V), C.byref(E), C.byref(wt)))
        self.V, self.E, self.weighted = V.value, E.value, bool(wt.value)

    @classmethod
    def from_edges(cls, V, src, dst, w=None) -> "Graph":
        s = np.ascontiguousarray(src, np.uint32)
        d = np.ascontiguousarray(dst, np.uint32)
        ww = None if w is None else np.ascontiguousarray(w, np.uint32)
        if len(s) != len(d) or (ww is not None and len(ww) != len(s)):
            raise ValueError("src, dst and w must have the same length")
        h = C.c_void_p()
        _check(lib().tg_graph_from_edges(V, len(s), s.ctypes.data_as(C.c_void_p),
                                         d.ctypes.data_as(C.c_void_p),
                                         None if ww is None else ww.ctypes.data_as(C.c_void_p),
                                         C.byref(h)))
        return cls(h)

    @classmethod
    def load_edge_list(cls, path, directed=True, weighted=False) -> "Graph":
        h = C.c_void_p()
        _check(lib().tg_graph_load_edge_list(os.fsencode(path), int(directed), int(weighted),
                                             C.byref(h)))
        return cls(h)

    def edges(self):
        src, dst = np.empty(self.E, np.uint32), np.empty(self.E, np.uint32)
        w = np.empty(self.E, np.uint32) if self.weighted else None
        _check(lib().tg_graph_edges(self.h, src.ctypes.data_as(C.c_void_p),
                                    dst.ctypes.data_as(C.c_void_p),
                                    None if w is None else w.ctypes.data_as(C.c_void_p)))
        return src, dst, w

    def close(self):
        if self.h:
            lib().tg_graph_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def tg_engine_create(graph: Graph, partitions=1, device=0, weighted=None, in_csr=True, rank=0, world=1,
                     comm=None, strategy=TG_PART_DEGREE, part_seed=4):
    if weighted is None:
        weighted = graph.weighted
    at = _attr(partitions, device, weighted, in_csr, rank, world, comm, strategy, part_seed)
    h = C.c_void_p()
    _check(lib().tg_engine_create(graph.h, C.byref(at), C.byref(h)))
    return h


def tg_partition_size(V: int, p: int, P: int) -> int:
    """|V_p| under the degree-serpentine deal (host only, no GPU needed)."""
    out = C.c_uint64()
    _check(lib().tg_partition_size(V, p, P, C.byref(out)))
    return out.value


def tg_engine_free(h) -> None:
    lib().tg_engine_free(h)


def tg_engine_info(h) -> dict:
    i = tg_info()
    _check(lib().tg_engine_info(h, C.byref(i)))
    return {f: getattr(i, f) for f, _ in tg_info._fields_}


def tg_engine_partition_info(h, p: int, P: int) -> dict:
    i = tg_part_info()
    slots = np.zeros(P, np.uint64)
    _check(lib().tg_engine_partition_info(h, p, C.byref(i), slots.ctypes.data_as(C.c_void_p)))
    d = {f: getattr(i, f) for f, _ in tg_part_info._fields_}
    d["slots_to"] = slots
    return d


def _out(out, V, dtype, device=None):
    """Output array -> (out, pointer, mem kind).  The library writes V elements
    of dtype's width, so a wrong width, a short, strided or foreign-device
    buffer is rejected here instead of being written out of bounds."""
    if out is None:
        out = np.empty(V, dtype)
    itemsize = np.dtype(dtype).itemsize
    if isinstance(out, np.ndarray):
        if out.dtype.itemsize != itemsize or out.dtype.kind != np.dtype(dtype).kind \
                or not out.flags.c_contiguous or out.size < V or not out.flags.writeable:
            raise ValueError(f"output must be a writeable contiguous {np.dtype(dtype)} array "
                             f"of length >= V ({V})")
        return out, out.ctypes.data_as(C.c_void_p), TG_MEM_HOST
    if hasattr(out, "data_ptr"):  # torch tensor (host or device)
        if out.element_size() != itemsize or out.numel() < V or not out.is_contiguous():
            raise ValueError(f"output tensor must be contiguous with {itemsize}-byte elements "
                             f"and >= V ({V}) elements")
        if getattr(out, "is_cuda", False):
            if device is not None and out.device.index != device:
                raise ValueError(f"output tensor on cuda:{out.device.index}, engine on cuda:{device}")
            return out, C.c_void_p(out.data_ptr()), TG_MEM_DEVICE
        return out, C.c_void_p(out.data_ptr()), TG_MEM_HOST
    raise TypeError("output must be a numpy array or a torch tensor")


def tg_bfs(h, V, source, out=None, device=None):
    out, ptr, mem = _out(out, V, np.uint32, device)
    st = tg_stats()
    _check(lib().tg_bfs(h, source, ptr, mem, C.byref(st)))
    return out, Stats.of(st)


def tg_sssp(h, V, source, out=None, device=None):
    out, ptr, mem = _out(out, V, np.uint32, device)
    st = tg_stats()
    _check(lib().tg_sssp(h, source, ptr, mem, C.byref(st)))
    return out, Stats.of(st)


def tg_pagerank(h, V, iterations=5, damping=0.85, out=None, device=None):
    out, ptr, mem = _out(out, V, np.float32, device)
    st = tg_stats()
    _check(lib().tg_pagerank(h, iterations, damping, ptr, mem, C.byref(st)))
    return out, Stats.of(st)


def tg_bc(h, V, sources, out=None, device=None):
    out, ptr, mem = _out(out, V, np.float64, device)
    s = np.ascontiguousarray(sources, np.uint64)
    st = tg_stats()
    _check(lib().tg_bc(h, s.ctypes.data_as(C.c_void_p), len(s), ptr, mem, C.byref(st)))
    return out, Stats.of(st)


def tg_cc(h, V, out=None, device=None):
    out, ptr, mem = _out(out, V, np.uint32, device)
    st = tg_stats()
    _check(lib().tg_cc(h, ptr, mem, C.byref(st)))
    return out, Stats.of(st)


def tg_engine_set_profiling(h, on: bool) -> None:
    _check(lib().tg_engine_set_profiling(h, int(on)))


TG_EXCHANGE_COPY, TG_EXCHANGE_FUSED = 0, 1
TG_PR_PUSH, TG_PR_PULL = 0, 1


def tg_engine_set_pagerank_comm(h, mode: int) -> None:
    _check(lib().tg_engine_set_pagerank_comm(h, int(mode)))


def tg_device_die_map(device: int = 0):
    """-> (ok, die_of numpy u8 per SM id) of the measured two-die map."""
    nsm, ok = C.c_int(0), C.c_int(0)
    _check(lib().tg_device_die_map(int(device), None, 0, C.byref(nsm), C.byref(ok)))
    out = np.zeros(max(nsm.value, 1), np.uint8)
    _check(lib().tg_device_die_map(int(device), out.ctypes.data_as(C.c_void_p), len(out),
                                   C.byref(nsm), C.byref(ok)))
    return bool(ok.value), out[:nsm.value]


def tg_engine_set_exchange(h, mode: int) -> None:
    _check(lib().tg_engine_set_exchange(h, int(mode)))


def tg_engine_kernel_stats(h) -> dict:
    """{kernel name: {launches, ms, algorithmic_bytes}} from the engine's ledger."""
    out = {}
    for kid in range(TG_K_COUNT):
        s = tg_kernel_stat()
        _check(lib().tg_engine_kernel_stat(h, kid, C.byref(s)))
        out[lib().tg_kernel_name(kid).decode()] = {
            "launches": s.launches, "ms": s.ms, "algorithmic_bytes": s.algorithmic_bytes}
    return out


class Engine:
    """Owning handle: a partitioned, device-resident graph."""

    def __init__(self, handle, comm=None, rank=0):
        self.h = handle
        self.comm = comm  # keeps the host-collective callbacks alive
        self.rank = rank
        inf = tg_engine_info(handle)
        self.V, self.E, self.P = inf["V"], inf["E"], inf["num_partitions"]
        self.device = inf["device"]
        self.info = inf

    @classmethod
    def from_edges(cls, V, src, dst, w=None, **kw) -> "Engine":
        return cls(tg_engine_create_edges(V, src, dst, w, **kw), kw.get("comm"), kw.get("rank", 0))

    @classmethod
    def from_graph(cls, graph: "Graph", **kw) -> "Engine":
        return cls(tg_engine_create(graph, **kw), kw.get("comm"), kw.get("rank", 0))

    @classmethod
    def rmat(cls, scale, **kw) -> "Engine":
        return cls(tg_engine_create_rmat(scale, **kw), kw.get("comm"), kw.get("rank", 0))

    def close(self):
        if self.h:
            tg_engine_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def partition_info(self, p):
        return tg_engine_partition_info(self.h, p, self.P)

    def bfs(self, source, out=None):
        return tg_bfs(self.h, self.V, source, out, self.device)

    def sssp(self, source, out=None):
        return tg_sssp(self.h, self.V, source, out, self.device)

    def pagerank(self, iterations=5, damping=0.85, out=None):
        return tg_pagerank(self.h, self.V, iterations, damping, out, self.device)

    def bc(self, sources, out=None):
        return tg_bc(self.h, self.V, sources, out, self.device)

    def cc(self, out=None):
        return tg_cc(self.h, self.V, out, self.device)

    def set_profiling(self, on=True):
        tg_engine_set_profiling(self.h, on)

    def kernel_stats(self):
        return tg_engine_kernel_stats(self.h)

    def set_pagerank_comm(self, mode):
        """TG_PR_PUSH (default) or TG_PR_PULL (tg_engine_set_pagerank_comm)."""
        tg_engine_set_pagerank_comm(self.h, mode)

    def set_async_collect(self, on=True):
        """tg_engine_set_async_collect: host outputs complete only after sync()."""
        _check(lib().tg_engine_set_async_collect(self.h, int(on)))

    def sync(self):
        """tg_engine_sync: wait for pending result copies."""
        _check(lib().tg_engine_sync(self.h))

    def last_ticket(self) -> int:
        """tg_engine_last_ticket: ticket of the latest asynchronous host collection."""
        t = C.c_uint64(0)
        _check(lib().tg_engine_last_ticket(self.h, C.byref(t)))
        return t.value

    def wait_ticket(self, ticket: int) -> None:
        """tg_engine_wait_ticket: collection `ticket` and all earlier are in host memory."""
        _check(lib().tg_engine_wait_ticket(self.h, int(ticket)))

    def set_exchange(self, mode):
        """TG_EXCHANGE_FUSED (default) or TG_EXCHANGE_COPY (tg_engine_set_exchange)."""
        tg_engine_set_exchange(self.h, mode)


class HostComm:
    """tg_hostcomm: the library's shared-memory node-local collective (the
    multi-process vote); created collectively over a TorchComm."""

    def __init__(self, comm: "TorchComm", rank: int, world: int):
        self.comm = comm
        self.h = C.c_void_p()
        _check(lib().tg_hostcomm_create(C.pointer(comm.struct), rank, world, C.byref(self.h)))

    def allreduce(self, vals, ops):
        d = np.ascontiguousarray(vals, np.uint64).copy()
        o = np.ascontiguousarray(ops, np.int32)
        _check(lib().tg_hostcomm_allreduce_u64(self.h, d.ctypes.data_as(C.c_void_p), len(d),
                                               o.ctypes.data_as(C.c_void_p)))
        return d

    def close(self):
        if self.h:
            lib().tg_hostcomm_free(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
