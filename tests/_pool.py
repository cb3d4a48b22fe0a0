"""Run oracle evaluations on all host cores (test infrastructure).

The oracle is plain single-threaded numpy; the large parity cases (config-5
sampled rows, long histories) split their independent pieces (row chunks,
elapsed times) over a process pool.  `spawn` workers: the parent holds a CUDA
context, the workers never touch CUDA.  Nothing here computes anything itself.
"""
from __future__ import annotations

import multiprocessing as mp
import os
from concurrent.futures import ProcessPoolExecutor

import numpy as np


def workers() -> int:
    return max(1, min(os.cpu_count() or 1, 32))


def _elastic_rows(args):
    from oracle import elastic as OE
    geom, G, nu, D, rows = args
    return OE.matvec_rows(geom, G, nu, D, rows)


def _poro_dense(args):
    from oracle import poro as OP
    geom, mat, tau = args
    return OP.assemble_dense(geom, mat, tau)


def _poro_row_blocks(args):
    from oracle import poro as OP
    geom, mat, tau, rows = args
    k = OP.constants(mat["G"], mat["nu"], mat["nu_u"], mat["alpha"], mat["kappa"])
    return np.stack([OP.row_blocks(geom, k, tau, int(i)) for i in rows])


def _map(fn, jobs):
    if len(jobs) == 1 or workers() == 1:
        return [fn(j) for j in jobs]
    with ProcessPoolExecutor(max_workers=min(workers(), len(jobs)),
                             mp_context=mp.get_context("spawn")) as ex:
        return list(ex.map(fn, jobs))


def elastic_rows(geom, G, nu, D, rows) -> np.ndarray:
    """oracle.elastic.matvec_rows over row chunks in parallel."""
    rows = np.asarray(rows)
    chunks = [c for c in np.array_split(rows, min(rows.size, 4 * workers())) if c.size]
    return np.concatenate(_map(_elastic_rows, [(geom, G, nu, D, c) for c in chunks]))


def poro_dense_many(geom, mat, taus) -> list:
    """oracle.poro.assemble_dense at each elapsed time, in parallel."""
    return _map(_poro_dense, [(geom, mat, float(t)) for t in taus])


def poro_row_blocks_many(geom, mat, taus, rows) -> list:
    """oracle.poro.row_blocks of the given target rows at each elapsed time:
    list over taus of [len(rows), N, 3, 3] (ABI convention)."""
    return _map(_poro_row_blocks, [(geom, mat, float(t), list(rows)) for t in taus])
