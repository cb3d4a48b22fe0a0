"""ctypes binding of libddm.so (include/ddm.h).  Argument marshalling only:
every step of the hot path runs inside the library's CUDA kernels.  There is
no CPU fallback — importing this module fails loudly if the library is
missing."""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
# DDM_LIB: alternative build of the same library (tuning experiments only)
LIB_PATH = os.environ.get("DDM_LIB") or os.path.join(_HERE, "libddm.so")

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; g.build()'` "
        "(there is no CPU fallback)")

lib = C.CDLL(LIB_PATH)

# status codes
OK, ERR_ARG, ERR_CUDA, ERR_NOCONV, ERR_NCCL, ERR_GEOM, ERR_OOM = range(7)
FMM, DIRECT, HIST_PERLAG = 0, 1, 2
GMRES_NO_PRECOND = 8
GMRES_PC_POINT = 32   # point-block Jacobi instead of the default leaf blocks
BBFMM = 16   # | n << 8: Chebyshev (bbFMM) far field with n nodes per dimension

TC = dict(N=0, CELLS=1, LEAVES=2, LEVELS=3, V=4, URANGES=5, NEAR_PAIRS=6, P2P_ITEMS=7,
          OWNED_LO=8, OWNED_HI=9, P=10, W=11, W_MIN=12, X=13, X_MIN=14, UXRANGES=15,
          NEAR_PAIRS_P2P=16)
NCOUNTS = 20
EX = dict(KEYS=0, PERM=1, ROOT=2, LEVEL=3, IX=4, IY=5, START=6, COUNT=7, PARENT=8,
          FIRST_CHILD=9, NCHILD=10, LEAF=11, V_OFF=12, V_IDX=13, LEAVES=14, U_OFF=15, U_LO=16,
          U_HI=17, W_OFF=18, W_IDX=19, X_OFF=20, X_IDX=21, UX_OFF=22, UX_LO=23, UX_HI=24)
STAGES = ["prep", "p2m", "m2m", "m2l", "l2l", "p2p", "final", "comm", "l2p", "p2l"]


class Material(C.Structure):
    _fields_ = [("kind", C.c_int), ("G", C.c_double), ("nu", C.c_double),
                ("nu_u", C.c_double), ("alpha", C.c_double), ("kappa", C.c_double)]


_vp = C.c_void_p
_dp = C.c_void_p          # device pointers are passed as integers
_i64 = C.c_int64
_d = C.c_double
_i = C.c_int


def _proto(name, res, *args):
    f = getattr(lib, name)
    f.restype = res
    f.argtypes = list(args)
    return f


ddm_version = _proto("ddm_version", C.c_char_p)
ddm_last_error = _proto("ddm_last_error", C.c_char_p, _vp)
ddm_nccl_unique_id = _proto("ddm_nccl_unique_id", _i, _vp)
ddm_ctx_create = _proto("ddm_ctx_create", _i, _i, _vp, _i, _i, C.POINTER(_vp))
ddm_ctx_destroy = _proto("ddm_ctx_destroy", None, _vp)
ddm_build_tree = _proto("ddm_build_tree", _i, _vp, _dp, _dp, _dp, _dp, _i64, _i, _i, _d, _vp,
                        C.POINTER(_vp))
ddm_tree_free = _proto("ddm_tree_free", None, _vp)
ddm_tree_counts = _proto("ddm_tree_counts", _i, _vp, C.POINTER(_i64))
ddm_tree_build_times = _proto("ddm_tree_build_times", _i, _vp, C.POINTER(C.c_double))
TB = ["keys", "sort", "cells", "lists", "sched", "total"]
ddm_tree_export = _proto("ddm_tree_export", _i, _vp, _i, _vp, _i64)
ddm_tree_partition = _proto("ddm_tree_partition", _i, _vp, _i, _i)
ddm_split_costs = _proto("ddm_split_costs", _i, C.POINTER(_i64), _i64, _i, _i, C.POINTER(_i))
ddm_matvec = _proto("ddm_matvec", _i, _vp, _vp, C.POINTER(Material), _d, _dp, _dp, _i, _vp)
ddm_shard_owner = _proto("ddm_shard_owner", _i, C.POINTER(_i), C.POINTER(_i), _i, C.POINTER(_i64), _i,
                          C.POINTER(_i))
ddm_matvec_sim = _proto("ddm_matvec_sim", _i, _vp, C.POINTER(_vp), _i, C.POINTER(Material), _dp,
                        _dp, _vp)
ddm_history_apply = _proto("ddm_history_apply", _i, _vp, _vp, C.POINTER(Material), _d, _i, _dp,
                           _dp, _i, _vp)
ddm_history_rhs = _proto("ddm_history_rhs", _i, _vp, _vp, C.POINTER(Material), _d, _i, _dp, _dp,
                         _dp, _i, _vp)
ddm_march_guess = _proto("ddm_march_guess", _i, _vp, _i, _dp, _i64, _i, _dp, _vp)
ddm_gmres_solve = _proto("ddm_gmres_solve", _i, _vp, _vp, C.POINTER(Material), _d, _dp, _dp, _d,
                         _i, _i, _i, C.POINTER(_i), C.POINTER(_d), _vp)
ddm_precond_apply = _proto("ddm_precond_apply", _i, _vp, _vp, C.POINTER(Material), _d, _dp, _dp,
                           _i, _vp)
ddm_farfield_rhs = _proto("ddm_farfield_rhs", _i, _vp, _dp, _i64, _i, _d, _d, _d, _i, _d, _dp,
                          _vp)
ddm_sif = _proto("ddm_sif", _i, _vp, _dp, _dp, _dp, _i, _d, _d, _dp, _dp, _vp)
ddm_tip_growth = _proto("ddm_tip_growth", _i, _vp, _i, _dp, _dp, _dp, _dp, _dp, _dp, _vp, _d,
                        _vp, _dp, _dp, _dp, _dp, _vp, _vp)
ddm_set_profiling = _proto("ddm_set_profiling", _i, _vp, _i)
ddm_stage_times = _proto("ddm_stage_times", _i, _vp, C.POINTER(_d))

EXPORTED = ["ddm_version", "ddm_last_error", "ddm_nccl_unique_id", "ddm_ctx_create",
            "ddm_ctx_destroy", "ddm_build_tree", "ddm_tree_free", "ddm_tree_counts",
            "ddm_tree_export", "ddm_tree_partition", "ddm_split_costs", "ddm_matvec", "ddm_matvec_sim", "ddm_shard_owner",
            "ddm_history_apply", "ddm_history_rhs", "ddm_march_guess", "ddm_gmres_solve", "ddm_precond_apply",
            "ddm_farfield_rhs", "ddm_sif", "ddm_tip_growth",
            "ddm_set_profiling", "ddm_stage_times", "ddm_tree_build_times"]
