"""Worker functions for the multi-process tests (spawned; must be importable)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def _init(rank, world, port):
    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    return dist


def comm_worker(rank, world, port):
    """Host collectives of the multi-process engine (tg_comm over gloo)."""
    import ctypes as C

    import torch

    import paper_1312_3018_b200 as tg

    dist = _init(rank, world, port)
    comm = tg.TorchComm()
    # allgather: rank r contributes bytes r, r+1, ... (variable content, fixed size)
    n = 37
    send = (np.arange(n, dtype=np.uint8) + rank).astype(np.uint8)
    recv = np.zeros(n * world, np.uint8)
    assert comm._ag(None, send.ctypes.data, recv.ctypes.data, n) == 0
    for r in range(world):
        assert np.array_equal(recv[r * n:(r + 1) * n], (np.arange(n) + r).astype(np.uint8))
    # allreduce sum and min, including the all-ones sentinel
    s = (C.c_uint64 * 3)(rank + 1, 1 << 40, (1 << 64) - 1)   # sums are modulo 2^64
    assert comm._ar(None, s, 3, 0) == 0
    assert s[0] == world * (world + 1) // 2 and s[1] == world << 40
    assert s[2] == ((1 << 64) - world) % (1 << 64)
    m = (C.c_uint64 * 2)((1 << 64) - 1, 100 + rank)
    assert comm._ar(None, m, 2, 1) == 0
    assert m[0] == (1 << 64) - 1 and m[1] == 100
    m2 = (C.c_uint64 * 1)((1 << 64) - 1 if rank else 7)
    assert comm._ar(None, m2, 1, 1) == 0 and m2[0] == 7
    # the partition plan, computed per rank on the host: sizes add up to V and
    # match the oracle's degree partition
    V = 1000 + world
    vp = tg.tg_partition_size(V, rank, world)
    t = torch.tensor([vp], dtype=torch.int64)
    dist.all_reduce(t)
    assert int(t.item()) == V
    if rank == 0:
        import oracle

        rng = np.random.default_rng(5)
        src = rng.integers(0, V, 8 * V).astype(np.uint32)
        dst = rng.integers(0, V, 8 * V).astype(np.uint32)
        part, _ = oracle.Graph(V, src, dst).partition(world)
        for p in range(world):
            assert tg.tg_partition_size(V, p, world) == int((part == p).sum())
    dist.barrier()
    dist.destroy_process_group()


def hostcomm_worker(rank, world, port):
    """The library's shared-memory collective (tg_hostcomm: the multi-process
    vote) against torch.distributed on the same values: sums mod 2^64, minima
    with the all-ones sentinel, mixed ops in one call, many epochs in a row
    (the two value buffers alternate), ranks arriving in skewed order."""
    import time

    import torch

    import paper_1312_3018_b200 as tg

    dist = _init(rank, world, port)
    comm = tg.TorchComm()
    hc = tg.HostComm(comm, rank, world)
    rng = np.random.default_rng(100 + rank)
    U64 = (1 << 64) - 1
    for it in range(300):
        n = 1 + it % 16
        vals = rng.integers(0, 1 << 62, n, dtype=np.uint64)
        if it % 7 == 0:
            vals[0] = U64
        ops = np.array([(it + i) % 2 for i in range(n)], np.int32)
        if it % 50 == rank:            # one rank arrives late
            time.sleep(0.02)
        got = hc.allreduce(vals, ops)
        allv = [torch.zeros(n, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allv, torch.from_numpy(vals.view(np.int64)))
        allv = [a.numpy().view(np.uint64) for a in allv]
        for i in range(n):
            col = [int(a[i]) for a in allv]
            want = min(col) if ops[i] == 1 else sum(col) % (1 << 64)
            assert int(got[i]) == want, (it, i, int(got[i]), want)
    hc.close()
    dist.barrier()
    dist.destroy_process_group()


def pr_pull(eng):
    """PageRank with ghost-pull communication (collective), then back to push."""
    import paper_1312_3018_b200 as tg

    eng.set_pagerank_comm(tg.TG_PR_PULL)
    r = eng.pagerank(5)[0]
    r = None if r is None else r.copy()
    eng.set_pagerank_comm(tg.TG_PR_PUSH)
    return r


def engine_worker(rank, world, port, scale, device, exchange=1, direction=None):
    """One partition per process on `device`; boundary messages through
    CUDA-IPC-mapped peer arenas (exchange 1: written by the compute kernels
    into the peers' arenas; 0: outbox + peer copies); rank 0 checks against
    the oracle.  direction: TG_DIRECTION for BFS / BC (None = auto)."""
    if direction:
        os.environ["TG_DIRECTION"] = direction
    if device < 0:  # one GPU per rank
        device = rank
    import inputs
    import paper_1312_3018_b200 as tg

    dist = _init(rank, world, port)
    comm = tg.TorchComm()
    src, dst, w = inputs.rmat_edges(scale, weights=True)
    V = 1 << scale
    eng_e = tg.Engine.from_edges(V, src, dst, w, rank=rank, world=world, comm=comm, device=device)
    eng_g = tg.Engine.rmat(scale, rank=rank, world=world, comm=comm, device=device)
    srcs = [int(x) for x in inputs.list_sources(src, 4)]
    results = []
    for eng in (eng_e, eng_g):
        # the fused transport was kept only after the peer self-test passed
        assert eng.info["peer_probe"] == 1 and eng.info["exchange"] == tg.TG_EXCHANGE_FUSED
        eng.set_exchange(exchange)
        pi = eng.partition_info(rank)
        assert pi["Vp"] == tg.tg_partition_size(V, rank, world)
        out = {"bfs": [eng.bfs(s)[0].copy() for s in srcs],
               "sssp": [eng.sssp(s)[0].copy() for s in srcs[:2]],
               "pr": eng.pagerank(5)[0].copy(),
               "pr_pull": pr_pull(eng),
               "bc": eng.bc(srcs[:2])[0].copy(),
               "cc": eng.cc()[0].copy()}
        results.append(out)
    if rank == 0:
        import oracle

        G = oracle.Graph(V, src, dst, w)
        for out in results:
            for s, lv in zip(srcs, out["bfs"]):
                assert np.array_equal(lv, G.bfs(s)), ("bfs", s)
            for s, d in zip(srcs[:2], out["sssp"]):
                assert np.array_equal(d, G.sssp(s)), ("sssp", s)
            ref = G.pagerank(5)
            assert (np.abs(out["pr"] - ref) / ref).max() <= 1e-5
            assert (np.abs(out["pr_pull"] - ref) / ref).max() <= 1e-5, "ghost-pull PageRank"
            bref = G.bc(srcs[:2])
            assert np.allclose(out["bc"], bref, rtol=1e-4, atol=1e-12 * max(1.0, bref.max()))
            assert np.array_equal(out["cc"], G.cc()), "cc"
    eng_e.close()
    eng_g.close()
    dist.barrier()
    dist.destroy_process_group()
