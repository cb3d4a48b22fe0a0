"""Test helpers: canonical forms of tree exports for bit-exact comparison."""
from __future__ import annotations

import numpy as np


def has_gpu() -> bool:
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def oracle_u_ranges(t, U: dict) -> dict:
    """Oracle U(B) (sets of leaves) -> merged sorted source-element ranges
    [lo, hi) in sorted order, keyed by leaf cell index."""
    out = {}
    for b, lst in U.items():
        rs = sorted((int(t.start[a]), int(t.start[a] + t.count[a])) for a in lst)
        merged = []
        for lo, hi in rs:
            if merged and merged[-1][1] == lo:
                merged[-1][1] = hi
            else:
                merged.append([lo, hi])
        out[b] = [tuple(r) for r in merged]
    return out


def gpu_u_ranges(tree, prefix="U") -> dict:
    """U ranges per leaf (prefix "UX": U minus the X lists)."""
    leaves = tree.export("LEAVES")
    off = tree.export(prefix + "_OFF")
    lo = tree.export(prefix + "_LO")
    hi = tree.export(prefix + "_HI")
    return {int(leaves[k]): [(int(lo[r]), int(hi[r])) for r in range(off[k], off[k + 1])]
            for k in range(leaves.size)}


def gpu_x_lists(tree) -> dict:
    """X lists per leaf as sorted canonical cell indices (the library keeps
    them in element order)."""
    leaves = tree.export("LEAVES")
    off = tree.export("X_OFF")
    idx = tree.export("X_IDX")
    return {int(leaves[k]): sorted(int(v) for v in idx[off[k]:off[k + 1]])
            for k in range(leaves.size)}


def gpu_v_lists(tree) -> dict:
    off = tree.export("V_OFF")
    idx = tree.export("V_IDX")
    return {c: [int(v) for v in idx[off[c]:off[c + 1]]] for c in range(off.size - 1)}


def rel_l2(a, b) -> float:
    a = np.asarray(a, dtype=np.float64).ravel()
    b = np.asarray(b, dtype=np.float64).ravel()
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb > 0 else 1.0))


def gpu_w_lists(tree) -> dict:
    leaves = tree.export("LEAVES")
    off = tree.export("W_OFF")
    idx = tree.export("W_IDX")
    return {int(leaves[k]): [int(v) for v in idx[off[k]:off[k + 1]]] for k in range(leaves.size)}
