"""BASELINE configs[4] (C5): RMAT-30 (2^30 vertices, 2^34 edges, the paper's
largest graph, Table 2) BFS + PageRank across 8 B200, one
process per GPU, with its checks:

* BFS from the bench's first source: exact streaming certificate over the
  regenerated 2^34-edge stream (oracle_bfs_cert_edges).
* PageRank (5 rounds): the oracle recomputes round 5 from the GPU's round-4
  ranks for a vertex sample (top in-degree hubs + random), 1e-5 relative, and
  the global mass identity (SURVEY 8(c) feasibility rule for s = 30).

Launch: python -m torch.distributed.run --nnodes=1 --nproc-per-node 8
        --master-addr 127.0.0.1 --master-port P scripts/c5_rmat30.py [--scale 30]
Prints one JSON line (rank 0) with GTEPS per algorithm, then "C5 OK".
"""
import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--scale", type=int, default=30)
    ap.add_argument("--sources", type=int, default=1)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dist.init_process_group("nccl")
    import inputs
    import paper_1312_3018_b200 as tg

    scale = args.scale
    V, E = 1 << scale, 16 << scale
    t0 = time.time()
    eng = tg.Engine.rmat(scale, weighted=False, in_csr=True, rank=rank, world=world,
                         comm=tg.TorchComm(), device=local)
    build_s = time.time() - t0
    srcs = [int(s) for s in inputs.rmat_sources(scale, args.sources)]
    res = {"bfs": [], "pagerank": None}
    lvs = []
    for s in srcs:
        lv, st = eng.bfs(s)
        res["bfs"].append({"source": s, "ms": st.device_ms, "supersteps": st.supersteps,
                           "gteps": st.traversed_edges / st.device_ms / 1e6})
        lvs.append(None if lv is None else lv.copy())
    r4, _ = eng.pagerank(4)
    r4 = None if r4 is None else r4.copy()
    r5, st = eng.pagerank(5)
    res["pagerank"] = {"ms_per_round": st.device_ms / 5, "gteps": st.traversed_edges / st.device_ms / 1e6}
    eng.close()
    ok = True
    if rank == 0:
        import oracle

        t1 = time.time()
        certs = [oracle.StreamingCertificate(V, s, lv, weighted=False) for s, lv in zip(srcs, lvs)]
        outdeg = np.zeros(V, np.uint32)
        indeg = np.zeros(V, np.uint32)
        chunk = 1 << 28
        for first in range(0, E, chunk):
            src, dst, _ = inputs.rmat_edges(scale, first=first, count=min(chunk, E - first))
            for c in certs:
                c.feed(src, dst)
            oracle.outdeg_edges(V, src, outdeg)
            oracle.outdeg_edges(V, dst, indeg)
        ok = all(c.holds() for c in certs)
        rng = np.random.default_rng(2024)
        sample = np.unique(np.concatenate([np.argsort(indeg)[-256:], rng.integers(0, V, 8192)]))
        mask = np.zeros((V + 63) // 64, np.uint64)
        np.bitwise_or.at(mask, sample >> 6, np.uint64(1) << (sample & 63).astype(np.uint64))
        slot = np.zeros(V, np.uint32)
        slot[sample] = np.arange(len(sample), dtype=np.uint32)
        acc = np.zeros(len(sample))
        for first in range(0, E, chunk):
            src, dst, _ = inputs.rmat_edges(scale, first=first, count=min(chunk, E - first))
            oracle.pr_sample_edges(V, src, dst, mask, slot, r4, outdeg, acc)
        d = 0.85
        pred = (1 - d) / V + d * acc
        rel = np.abs(r5[sample].astype(np.float64) - pred) / pred
        mass_pred = (1 - d) + d * r4[outdeg > 0].astype(np.float64).sum()
        mass_ok = abs(r5.astype(np.float64).sum() - mass_pred) <= 1e-5 * mass_pred
        ok = ok and rel.max() <= 1e-5 and mass_ok
        res.update({"scale": scale, "gpus": world, "build_s": build_s, "bfs_certificates": ok,
                    "pr_sample_max_rel": float(rel.max()), "pr_mass_ok": bool(mass_ok),
                    "host_check_s": time.time() - t1})
        print(json.dumps(res), flush=True)
        print("C5 OK" if ok else "C5 FAILED", flush=True)
    flag = torch.tensor([1 if ok else 0], device="cuda")
    dist.all_reduce(flag, op=dist.ReduceOp.MIN)
    dist.destroy_process_group()
    return 0 if int(flag.item()) else 1


if __name__ == "__main__":
    sys.exit(main())
