"""B200-native FMM displacement-discontinuity matvec (arXiv 1812.05087).

The hot path (tree build, P2M/M2M/M2L/L2L/L2P, near-field P2P, GMRES, SIF)
lives in libddm.so (hand-written fp64 CUDA for sm_100a, C-ABI in
include/ddm.h).  This package is its argument-marshalling binding; importing it
fails if the library has not been built (no CPU fallback).
"""
from . import _lib  # noqa: F401  (raises ImportError if libddm.so is missing)
from .api import (  # noqa: F401
    Context,
    DDMError,
    NoConvergence,
    Tree,
    farfield_rhs,
    gmres_solve,
    history_apply,
    history_rhs,
    march_guess,
    material,
    material_from_dict,
    matvec,
    matvec_sim,
    nccl_unique_id,
    precond_apply,
    sif,
    shard_owner,
    split_costs,
    tip_growth,
)

from .march import march  # noqa: F401,E402
from .propagate import propagate  # noqa: F401,E402

__version__ = "0.1.0"
