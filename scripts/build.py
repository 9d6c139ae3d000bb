"""Build helpers for the three native pieces of the repo.

* inputs/libtginputs.so  -- seeded input generator (host, gcc)
* oracle/liboracle.so    -- CPU oracle (host, gcc, single-threaded, -O2); test infrastructure
* paper_1312_3018_b200/libtgraph.so -- the CUDA product library (nvcc, sm_100a)

Everything is built in-tree so the .so files travel to the GPU box with gpurun.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
INPUTS_SO = os.path.join(ROOT, "inputs", "libtginputs.so")
ORACLE_SO = os.path.join(ROOT, "oracle", "liboracle.so")
TGRAPH_SO = os.path.join(ROOT, "paper_1312_3018_b200", "libtgraph.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _stale(target: str, sources: list[str]) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd: list[str]) -> None:
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout + r.stderr)
        raise RuntimeError(f"build failed: {cmd[0]} -> exit {r.returncode}")


def build_inputs(force: bool = False) -> str:
    srcs = [os.path.join(ROOT, "inputs", f) for f in ("tg_inputs.c", "tg_inputs.h")]
    if force or _stale(INPUTS_SO, srcs):
        _run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=c99", "-o", INPUTS_SO, srcs[0]])
    return INPUTS_SO


def build_oracle(force: bool = False) -> str:
    srcs = [os.path.join(ROOT, "oracle", f) for f in ("oracle.c", "oracle.h")]
    if force or _stale(ORACLE_SO, srcs):
        _run(["gcc", "-O2", "-fopenmp", "-fPIC", "-shared", "-std=gnu99", "-o", ORACLE_SO, srcs[0]])
    return ORACLE_SO


def _nccl_dirs() -> tuple[str | None, str | None]:
    try:
        import nvidia.nccl  # type: ignore

        base = list(nvidia.nccl.__path__)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    except Exception:
        pass
    return None, None


def build_tgraph(force: bool = False) -> str:
    """Each .cu compiles to build/<name>.o in parallel (a file is recompiled when
    it or any header is newer than its object), then one nvcc link -> .so."""
    from concurrent.futures import ThreadPoolExecutor

    csrc = os.path.join(ROOT, "paper_1312_3018_b200", "csrc")
    cu = sorted(glob.glob(os.path.join(csrc, "*.cu")))
    headers = sorted(glob.glob(os.path.join(csrc, "*.cuh"))) + \
        sorted(glob.glob(os.path.join(csrc, "*.h"))) + [
        os.path.join(ROOT, "include", "tgraph.h"),
        os.path.join(ROOT, "inputs", "tg_inputs.h"),
    ]
    if not (force or _stale(TGRAPH_SO, cu + headers)):
        return TGRAPH_SO
    obj_dir = os.path.join(ROOT, "build", "tgraph")
    os.makedirs(obj_dir, exist_ok=True)
    flags = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
             "-Xptxas", "-v", "--expt-relaxed-constexpr",
             "-I", os.path.join(ROOT, "include"), "-I", os.path.join(ROOT, "inputs")]

    def compile_one(src):
        obj = os.path.join(obj_dir, os.path.basename(src)[:-3] + ".o")
        if force or _stale(obj, [src] + headers):
            r = subprocess.run([NVCC, *flags, "-c", "-o", obj, src], cwd=ROOT, capture_output=True,
                               text=True)
            if r.returncode != 0:
                return obj, r.stdout + r.stderr, False
            with open(obj + ".ptxas.log", "w") as f:
                f.write(r.stderr)
        return obj, "", True

    with ThreadPoolExecutor(max_workers=min(len(cu), os.cpu_count() or 4)) as ex:
        res = list(ex.map(compile_one, cu))
    bad = [(o, log) for o, log, ok in res if not ok]
    if bad:
        for o, log in bad:
            sys.stderr.write(f"{o}:\n{log}\n")
        raise RuntimeError("nvcc failed")
    objs = [o for o, _, _ in res]
    r = subprocess.run([NVCC, *ARCH, "-shared", "-o", TGRAPH_SO, *objs], cwd=ROOT,
                       capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc link failed")
    with open(os.path.join(ROOT, "build_ptxas.log"), "w") as f:
        for o in objs:
            f.write(open(o + ".ptxas.log").read() if os.path.exists(o + ".ptxas.log") else "")
    return TGRAPH_SO


def build_all(force: bool = False) -> None:
    build_inputs(force)
    build_oracle(force)
    build_tgraph(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print("built:", INPUTS_SO, ORACLE_SO, TGRAPH_SO)
