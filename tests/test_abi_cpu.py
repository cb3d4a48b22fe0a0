"""CPU-side checks of the C-ABI library: it loads, exports every symbol
include/ddm.h declares, and its host-only partition helper is correct."""
import ctypes
import os
import re
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1812_05087_b200", "libddm.so")


@pytest.fixture(scope="module")
def built():
    from paper_1812_05087_b200 import build as B
    B.build()
    return LIB


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "ddm.h")).read()
    return sorted(set(re.findall(r"\b(ddm_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol(built):
    lib = ctypes.CDLL(built)
    syms = declared_symbols()
    assert len(syms) >= 18
    for s in syms:
        assert hasattr(lib, s), s
    out = subprocess.run(["nm", "-D", "--defined-only", built], capture_output=True, text=True).stdout
    for s in syms:
        assert re.search(rf"\bT {s}$", out, re.M), s


def test_library_is_sm100a(built):
    out = subprocess.run(["cuobjdump", "--list-elf", built], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_binding_marshals_names(built):
    import paper_1812_05087_b200 as D
    from paper_1812_05087_b200 import _lib
    assert set(_lib.EXPORTED) <= set(declared_symbols())
    assert D._lib.ddm_version().decode().startswith("ddm-b200")


def test_split_costs_host_logic(built):
    import paper_1812_05087_b200 as D
    rng = np.random.default_rng(0)
    for world in (1, 2, 3, 8):
        cost = rng.integers(0, 1000, 500).astype(np.int64)
        cost[100] = 200000            # one heavy leaf
        pre = np.concatenate([[0], np.cumsum(cost)[:-1]])
        tot = int(cost.sum())
        sp = D.split_costs(pre, tot, world)
        assert sp[0] == 0 and sp[-1] == 500 and np.all(np.diff(sp) >= 0)
        # rank r owns the leaves whose prefix lies in [r T/w, (r+1) T/w)
        for k in range(500):
            r = np.searchsorted(sp, k, side="right") - 1
            assert r * tot / world <= pre[k] + 1e-9 or r == 0
            assert pre[k] < (r + 1) * tot / world or r == world - 1
