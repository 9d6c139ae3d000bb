"""CPU-side checks of the C-ABI boundary: the library loads, exports every
symbol include/tgraph.h declares, and validates arguments before touching the
GPU.  No compute calls (there is no GPU here)."""
import ctypes as C
import os
import re
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "tgraph.h")


def declared_functions():
    txt = open(HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"^\s*(?:const\s+)?\w+\s*\*?\s*(tg_\w+)\s*\(", txt, flags=re.M)))


@pytest.fixture(scope="module")
def tglib():
    import sys

    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    from build import build_tgraph

    build_tgraph()
    from paper_1312_3018_b200 import tgraph

    return tgraph.lib()


def test_header_declares_the_boundary():
    fns = declared_functions()
    for f in ("tg_engine_create_edges", "tg_engine_create_rmat", "tg_engine_free", "tg_bfs",
              "tg_sssp", "tg_pagerank", "tg_bc", "tg_last_error", "tg_version"):
        assert f in fns


def test_library_exports_every_declared_symbol(tglib):
    so = os.path.join(ROOT, "paper_1312_3018_b200", "libtgraph.so")
    out = subprocess.run(["nm", "-D", "--defined-only", so], capture_output=True, text=True).stdout
    exported = set(re.findall(r"\s[TW]\s+(\w+)$", out, flags=re.M))
    missing = [f for f in declared_functions() if f not in exported]
    assert not missing, missing
    assert b"sm_100a" in tglib.tg_version()


def test_library_is_sm100a_only():
    so = os.path.join(ROOT, "paper_1312_3018_b200", "libtgraph.so")
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", so], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_argument_validation_precedes_cuda(tglib):
    from paper_1312_3018_b200 import tgraph

    with pytest.raises(tgraph.TGraphError) as e:
        tgraph.tg_engine_create_rmat(10, a=0.6, b=0.3, c=0.3)   # a+b+c > 1
    assert e.value.code == tgraph.TG_EINVAL
    with pytest.raises(tgraph.TGraphError) as e:
        tgraph.tg_engine_create_rmat(0)
    assert e.value.code == tgraph.TG_EINVAL
    with pytest.raises(tgraph.TGraphError) as e:
        tgraph.tg_engine_create_edges(0, [], [])
    assert e.value.code == tgraph.TG_EINVAL
    assert tglib.tg_bfs(None, 0, None, 0, None) == tgraph.TG_EINVAL
    assert tglib.tg_engine_set_exchange(None, tgraph.TG_EXCHANGE_FUSED) == tgraph.TG_EINVAL
    assert tglib.tg_engine_set_pagerank_comm(None, tgraph.TG_PR_PULL) == tgraph.TG_EINVAL
    assert tglib.tg_device_die_map(0, None, 0, None, None) == tgraph.TG_EINVAL
    assert tglib.tg_engine_last_ticket(None, None) == tgraph.TG_EINVAL
    assert tglib.tg_engine_wait_ticket(None, 0) == tgraph.TG_EINVAL
    assert b"NULL" in tglib.tg_last_error()


def test_product_package_never_imports_the_oracle():
    pkg = os.path.join(ROOT, "paper_1312_3018_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h")):
                src = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in src and "oracle.h" not in src, f
                assert "liboracle" not in src, f
