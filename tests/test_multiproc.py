"""Multi-process (one partition per process) paths.

CPU (gloo, world 2 and 3): the host collectives the library calls through
tg_comm (allgather of metadata, vote sums / minima, the all-ones sentinel) and
the per-rank partition plan against the oracle.
GPU: 2 and 3 processes on one B200 (cuda:0), one partition each, boundary
messages copied into CUDA-IPC-mapped peer arenas, or (fused exchange) written
there by the compute kernels -- the same code paths that cross NVLink between
GPUs -- checked against the oracle on rank 0."""
import socket

import pytest
import torch.multiprocessing as mp

import mp_workers


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("world", [2, 3])
def test_host_collectives_and_plan_gloo(world):
    mp.spawn(mp_workers.comm_worker, args=(world, _port()), nprocs=world, join=True)


@pytest.mark.parametrize("world", [2, 4])
def test_shared_memory_vote_gloo(world):
    mp.spawn(mp_workers.hostcomm_worker, args=(world, _port()), nprocs=world, join=True)


@pytest.mark.gpu
@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("exchange", [0, 1])
def test_ipc_partitions_on_one_gpu(world, exchange):
    mp.spawn(mp_workers.engine_worker, args=(world, _port(), 12, 0, exchange), nprocs=world,
             join=True)


@pytest.mark.gpu
@pytest.mark.parametrize("world,scale,direction", [(4, 18, "bottom"), (4, 18, None),
                                                   (8, 18, None), (8, 14, "top")])
def test_ipc_partitions_on_one_gpu_wide(world, scale, direction):
    """4 and 8 processes (one partition each) on one GPU at RMAT-18, fused
    exchange, direction-optimized BFS / BC across processes (forced bottom-up /
    pull-sigma, automatic, and top-down only), all five algorithms vs the
    oracle; the per-superstep vote runs in the library's shared-memory
    collective."""
    mp.spawn(mp_workers.engine_worker, args=(world, _port(), scale, 0, 1, direction),
             nprocs=world, join=True)
