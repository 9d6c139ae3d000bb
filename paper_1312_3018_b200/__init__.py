"""B200-native BSP graph superstep engine (TOTEM hot path, arXiv 1312.3018).

Thin ctypes binding of libtgraph.so (include/tgraph.h): argument marshalling
only -- every step of every algorithm runs in the CUDA kernels of csrc/.  There
is no CPU fallback: if the library is missing the import fails loudly.
"""
from .tgraph import (  # noqa: F401
    TG_EXCHANGE_COPY,
    TG_EXCHANGE_FUSED,
    TG_INF32,
    TG_PR_PULL,
    TG_PR_PUSH,
    TG_PART_DEGREE,
    TG_PART_RANDOM,
    TG_MEM_DEVICE,
    TG_MEM_HOST,
    Engine,
    Graph,
    Stats,
    TGraphError,
    TorchComm,
    HostComm,
    tg_partition_size,
    lib,
    tg_bc,
    tg_cc,
    tg_bfs,
    tg_engine_create,
    tg_engine_create_edges,
    tg_engine_create_rmat,
    tg_engine_free,
    tg_engine_info,
    tg_engine_partition_info,
    tg_engine_set_exchange,
    tg_engine_set_pagerank_comm,
    tg_device_die_map,
    tg_pagerank,
    tg_rmat_edges,
    tg_sssp,
)
