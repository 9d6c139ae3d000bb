"""Several GPUs (skipped on a box with fewer): one process per GPU, the fused
transport's peer stores / atomics crossing NVLink between distinct devices,
both exchange modes, all five algorithms against the oracle on rank 0
(the distinct-GPU peer-atomics path must be exercised before it is
relied on; the setup self-test asserted by the worker proves it per run).
TG_C5=1 on an 8-GPU box also runs BASELINE configs[4] (RMAT-30 BFS + PageRank
across 8 B200) with its checks, via scripts/c5_rmat30.py."""
import os
import socket
import subprocess
import sys

import pytest
import torch
import torch.multiprocessing as mp

import mp_workers

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NDEV = torch.cuda.device_count() if torch.cuda.is_available() else 0
pytestmark = [pytest.mark.gpu,
              pytest.mark.skipif(NDEV < 2, reason=f"needs >= 2 GPUs (this box has {NDEV})")]


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


@pytest.mark.parametrize("exchange", [0, 1])
def test_one_process_per_gpu(exchange):
    world = min(NDEV, 8)
    mp.spawn(mp_workers.engine_worker, args=(world, _port(), 16, -1, exchange, None), nprocs=world,
             join=True)


@pytest.mark.skipif(NDEV < 8 or os.environ.get("TG_C5") != "1",
                    reason="RMAT-30 across 8 B200 (C5): TG_C5=1 on an 8-GPU box")
def test_c5_rmat30_eight_gpus():
    r = subprocess.run([sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                        "--nproc-per-node", "8", "--master-addr", "127.0.0.1", "--master-port",
                        str(_port()), os.path.join(ROOT, "scripts", "c5_rmat30.py")],
                       cwd=ROOT, capture_output=True, text=True, timeout=7200)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "C5 OK" in r.stdout, r.stdout[-3000:]
