"""Run independent oracle jobs in forked children (test infrastructure).

Each job is a zero-argument callable; the children inherit the parent's arrays
(the oracle's CSR, the GPU results to compare) copy-on-write, so nothing large
is pickled, and each oracle call stays single-threaded -- several of them just
run side by side on the box's cores.  Jobs return small picklable values."""
import multiprocessing as mp
import os

_JOBS = None


def _run(i):
    return _JOBS[i]()


def fork_map(jobs, procs=None):
    global _JOBS
    _JOBS = list(jobs)
    if not _JOBS:
        return []
    n = procs or min(len(_JOBS), os.cpu_count() or 1)
    ctx = mp.get_context("fork")
    try:
        with ctx.Pool(n) as pool:
            return pool.map(_run, range(len(_JOBS)), chunksize=1)
    finally:
        _JOBS = None
