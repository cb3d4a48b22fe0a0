"""Thin Python face of the C-ABI (same names as include/ddm.h).  torch supplies
device memory, streams and the process-group bootstrap; all computation is in
libddm.so.  Errors raise DDMError with the library's message."""
from __future__ import annotations

import ctypes as C

import numpy as np
import torch

from . import _lib as L


class DDMError(RuntimeError):
    def __init__(self, code, msg):
        super().__init__(f"ddm error {code}: {msg}")
        self.code = code


class NoConvergence(DDMError):
    pass


def _stream_ptr(stream):
    if stream is None:
        stream = torch.cuda.current_stream()
    return C.c_void_p(stream.cuda_stream)


def _dev(t: torch.Tensor, name: str, dtype=torch.float64) -> int:
    if not isinstance(t, torch.Tensor) or not t.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if t.dtype != dtype:
        raise TypeError(f"{name} must be {dtype}")
    if not t.is_contiguous():
        raise TypeError(f"{name} must be contiguous")
    return t.data_ptr()


def material(kind=0, G=8e9, nu=0.25, nu_u=None, alpha=0.0, kappa=0.0) -> L.Material:
    return L.Material(int(kind), float(G), float(nu), float(nu if nu_u is None else nu_u),
                      float(alpha), float(kappa))


def material_from_dict(m: dict) -> L.Material:
    return material(m["kind"], m["G"], m["nu"], m.get("nu_u"), m.get("alpha", 0.0),
                    m.get("kappa", 0.0))


class Context:
    """One per process/GPU.  world > 1 needs an ncclUniqueId (bytes) that
    rank 0 made with nccl_unique_id() and broadcast via torch.distributed."""

    def __init__(self, device: int = 0, rank: int = 0, world: int = 1, nccl_uid: bytes | None = None):
        torch.cuda.set_device(device)
        h = C.c_void_p()
        uid = None
        if nccl_uid is not None:
            uid = C.create_string_buffer(bytes(nccl_uid), 128)
        rc = L.ddm_ctx_create(device, uid, rank, world, C.byref(h))
        self._h = h
        self.device, self.rank, self.world = device, rank, world
        if rc != L.OK:
            msg = L.ddm_last_error(h).decode() if h.value else ""
            raise DDMError(rc, msg)

    def check(self, rc):
        if rc == L.OK:
            return
        msg = L.ddm_last_error(self._h).decode()
        if rc == L.ERR_NOCONV:
            raise NoConvergence(rc, msg)
        raise DDMError(rc, msg)

    def close(self):
        if self._h and self._h.value:
            L.ddm_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def set_profiling(self, on: bool = True, serial: bool = False):
        """Per-stage CUDA events; serial=True also runs every stage on the
        caller's stream one after another (clean per-kernel durations)."""
        self.check(L.ddm_set_profiling(self._h, (2 if serial else 1) if on else 0))

    def stage_times(self) -> dict:
        arr = (C.c_double * len(L.STAGES))()
        self.check(L.ddm_stage_times(self._h, arr))
        return dict(zip(L.STAGES, list(arr)))


def nccl_unique_id() -> bytes:
    buf = C.create_string_buffer(128)
    rc = L.ddm_nccl_unique_id(buf)
    if rc != L.OK:
        raise DDMError(rc, "ncclGetUniqueId failed")
    return buf.raw


class Tree:
    """ddm_build_tree: geometry tensors on the device (float64, user order)."""

    def __init__(self, ctx: Context, xc, yc, half_len, beta, leaf_size: int = 32,
                 order_p: int = 20, min_leaf_side: float = 0.0, stream=None):
        self.ctx = ctx
        n = xc.numel()
        h = C.c_void_p()
        ctx.check(L.ddm_build_tree(ctx._h, _dev(xc, "xc"), _dev(yc, "yc"),
                                   _dev(half_len, "half_len"), _dev(beta, "beta"), n,
                                   int(leaf_size), int(order_p), float(min_leaf_side),
                                   _stream_ptr(stream), C.byref(h)))
        self._h = h
        self.n = n
        self.beta = beta
        self.counts = self._counts()

    def _counts(self) -> dict:
        arr = (C.c_int64 * L.NCOUNTS)()
        self.ctx.check(L.ddm_tree_counts(self._h, arr))
        return {k: int(arr[v]) for k, v in L.TC.items()}

    def build_times(self) -> dict:
        """ddm_tree_build_times: ms per build stage (keys, sort, cells, lists,
        sched) and the host wall time of the build call (total)."""
        arr = (C.c_double * len(L.TB))()
        self.ctx.check(L.ddm_tree_build_times(self._h, arr))
        return {k: float(arr[i]) for i, k in enumerate(L.TB)}

    def export(self, what: str) -> np.ndarray:
        c = self.counts
        n, nc, nl = c["N"], c["CELLS"], c["LEAVES"]
        spec = {"KEYS": (np.uint64, n), "PERM": (np.int32, n), "ROOT": (np.float64, 3),
                "V_OFF": (np.int32, nc + 1), "V_IDX": (np.int32, c["V"]),
                "LEAVES": (np.int32, nl), "U_OFF": (np.int32, nl + 1),
                "U_LO": (np.int32, c["URANGES"]), "U_HI": (np.int32, c["URANGES"]),
                "W_OFF": (np.int32, nl + 1), "W_IDX": (np.int32, c["W"]),
                "X_OFF": (np.int32, nl + 1), "X_IDX": (np.int32, c["X"]),
                "UX_OFF": (np.int32, nl + 1), "UX_LO": (np.int32, c["UXRANGES"]),
                "UX_HI": (np.int32, c["UXRANGES"])}
        dt, size = spec.get(what, (np.int32, nc))
        out = np.empty(max(size, 1), dtype=dt)
        self.ctx.check(L.ddm_tree_export(self._h, L.EX[what], out.ctypes.data_as(C.c_void_p),
                                         out.nbytes))
        return out[:size]

    def partition(self, rank: int, world: int):
        self.ctx.check(L.ddm_tree_partition(self._h, rank, world))
        self.counts = self._counts()

    def free(self):
        if self._h and self._h.value:
            L.ddm_tree_free(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


def _mode(mode) -> int:
    """"fmm" (complex-variable series), "direct", "perlag" (history), or
    "bbfmm<n>" (the paper's Chebyshev far field with n nodes per dimension,
    e.g. "bbfmm3", "bbfmm6"; elastic)."""
    if not isinstance(mode, str):
        return int(mode)
    if mode.startswith("bbfmm"):
        return L.BBFMM | (int(mode[5:]) << 8)
    return {"fmm": L.FMM, "direct": L.DIRECT, "perlag": L.HIST_PERLAG}[mode]


def matvec(ctx: Context, tree: Tree, mat, D: torch.Tensor, y: torch.Tensor | None = None,
           mode="fmm", elapsed: float = 0.0, stream=None) -> torch.Tensor:
    """ddm_matvec: y = A D, D [n, ncomp] float64 on the device, user order."""
    if y is None:
        y = torch.empty_like(D)
    ctx.check(L.ddm_matvec(ctx._h, tree._h, C.byref(mat), float(elapsed), _dev(D, "D"),
                           _dev(y, "y"), _mode(mode), _stream_ptr(stream)))
    return y


def matvec_sim(ctx: Context, trees, mat, D: torch.Tensor, y: torch.Tensor | None = None,
               stream=None) -> torch.Tensor:
    """ddm_matvec_sim: the sharded multi-rank elastic FMM matvec emulated on one
    device; trees[r] is the geometry partitioned as rank r of len(trees)."""
    if y is None:
        y = torch.empty_like(D)
    arr = (C.c_void_p * len(trees))(*[t._h.value for t in trees])
    ctx.check(L.ddm_matvec_sim(ctx._h, arr, len(trees), C.byref(mat), _dev(D, "D"), _dev(y, "y"),
                               _stream_ptr(stream)))
    return y


def history_apply(ctx, tree, mat, dt: float, D_hist: torch.Tensor, r: torch.Tensor | None = None,
                  mode="fmm", stream=None) -> torch.Tensor:
    """ddm_history_apply: r = sum_{m=1}^{h} A^(m) D^(h-m); D_hist [h, n, 3].
    mode "fmm" = fast form (one far pass + multi-lag near field), "perlag" =
    one FMM matvec per lag (the paper's scheme), "direct" = exact per lag."""
    h = D_hist.shape[0]
    if r is None:
        r = torch.empty((tree.n, 3), dtype=torch.float64, device=D_hist.device)
    ptr = _dev(D_hist, "D_hist") if h > 0 else 0
    ctx.check(L.ddm_history_apply(ctx._h, tree._h, C.byref(mat), float(dt), int(h), ptr,
                                  _dev(r, "r"), _mode(mode), _stream_ptr(stream)))
    return r


def history_rhs(ctx, tree, mat, dt: float, D_hist: torch.Tensor, b: torch.Tensor,
                rhs: torch.Tensor | None = None, mode="fmm", stream=None) -> torch.Tensor:
    """ddm_history_rhs: rhs = b - sum_{m=1}^{h} A^(m) D^(h-m)."""
    h = D_hist.shape[0]
    if rhs is None:
        rhs = torch.empty_like(b)
    ptr = _dev(D_hist, "D_hist") if h > 0 else 0
    ctx.check(L.ddm_history_rhs(ctx._h, tree._h, C.byref(mat), float(dt), int(h), ptr,
                                _dev(b, "b"), _dev(rhs, "rhs"), _mode(mode), _stream_ptr(stream)))
    return rhs


def march_guess(ctx, D_hist: torch.Tensor, order: int, x: torch.Tensor, stream=None) -> torch.Tensor:
    """ddm_march_guess: x = polynomial extrapolation (order <= 5) of the last
    solutions in D_hist [h, ...] (h = 0 -> x = 0)."""
    h = D_hist.shape[0]
    ptr = _dev(D_hist, "D_hist") if h > 0 else 0
    ctx.check(L.ddm_march_guess(ctx._h, int(h), ptr, int(x.numel()), int(order), _dev(x, "x"),
                                _stream_ptr(stream)))
    return x


def _pc_flags(precond) -> int:
    if precond is None or precond is False:
        return L.GMRES_NO_PRECOND
    if precond is True or precond == "leaf":
        return 0
    if precond == "point":
        return L.GMRES_PC_POINT
    raise ValueError(f"precond must be 'leaf', 'point' or False, not {precond!r}")


def precond_apply(ctx, tree, mat, x: torch.Tensor, y: torch.Tensor | None = None, dt: float = 0.0,
                  kind="leaf", stream=None) -> torch.Tensor:
    """ddm_precond_apply: y = M^-1 x for the GMRES preconditioner ("leaf" or
    "point" block Jacobi), user order."""
    if y is None:
        y = torch.empty_like(x)
    ctx.check(L.ddm_precond_apply(ctx._h, tree._h, C.byref(mat), float(dt), _dev(x, "x"),
                                  _dev(y, "y"), {"point": 1, "leaf": 2}[kind],
                                  _stream_ptr(stream)))
    return y


def gmres_solve(ctx, tree, mat, b: torch.Tensor, x: torch.Tensor | None = None, dt: float = 0.0,
                tol: float = 1e-10, restart: int = 2000, max_iter: int = 10000, mode="fmm",
                stream=None, raise_noconv: bool = True, precond="leaf"):
    """ddm_gmres_solve: returns (x, iters, rel_resid).  precond: right
    preconditioning by block Jacobi -- "leaf" (or True, default): inverse dense
    blocks of <= 32 consecutive elements of one leaf; "point": inverse element
    self blocks; False / None: plain GMRES."""
    if x is None:
        x = torch.zeros_like(b)
    it = C.c_int(0)
    rr = C.c_double(0.0)
    rc = L.ddm_gmres_solve(ctx._h, tree._h, C.byref(mat), float(dt), _dev(b, "b"), _dev(x, "x"),
                           float(tol), int(restart), int(max_iter),
                           _mode(mode) | _pc_flags(precond), C.byref(it),
                           C.byref(rr), _stream_ptr(stream))
    if rc == L.ERR_NOCONV and not raise_noconv:
        return x, it.value, rr.value
    ctx.check(rc)
    return x, it.value, rr.value


def farfield_rhs(ctx, beta: torch.Tensor, ncomp: int, p_f: float, sH: float, sh: float,
                 net: bool = False, b_p: float = 0.0, stream=None) -> torch.Tensor:
    n = beta.numel()
    b = torch.empty((n, ncomp), dtype=torch.float64, device=beta.device)
    ctx.check(L.ddm_farfield_rhs(ctx._h, _dev(beta, "beta"), n, int(ncomp), float(p_f), float(sH),
                                 float(sh), 1 if net else 0, float(b_p), _dev(b, "b"),
                                 _stream_ptr(stream)))
    return b


def sif(ctx, w_tip: torch.Tensor, ds_tip: torch.Tensor, a_tip: torch.Tensor, E: float, nu: float,
        stream=None):
    """ddm_sif (Olson, Eq.(SIF)): returns (K_I, K_II) device tensors."""
    n = w_tip.numel()
    KI = torch.empty_like(w_tip)
    KII = torch.empty_like(w_tip)
    ctx.check(L.ddm_sif(ctx._h, _dev(w_tip, "w_tip"), _dev(ds_tip, "ds_tip"), _dev(a_tip, "a_tip"),
                        int(n), float(E), float(nu), _dev(KI, "KI"), _dev(KII, "KII"),
                        _stream_ptr(stream)))
    return KI, KII


def tip_growth(ctx, KI: torch.Tensor, KII: torch.Tensor, x: torch.Tensor, y: torch.Tensor,
               a: torch.Tensor, beta: torch.Tensor, end: torch.Tensor, K_IC: float, stream=None):
    """ddm_tip_growth (Fig. 8 branch, reading R23): per tip, grow flag
    and the new element (x, y, a, beta, outward end) of the tips that grow."""
    n = KI.numel()
    grow = torch.empty(n, dtype=torch.int32, device=KI.device)
    ne = torch.empty(n, dtype=torch.int32, device=KI.device)
    nx, ny, na, nb = (torch.empty_like(KI) for _ in range(4))
    ctx.check(L.ddm_tip_growth(ctx._h, int(n), _dev(KI, "KI"), _dev(KII, "KII"), _dev(x, "x"),
                               _dev(y, "y"), _dev(a, "a"), _dev(beta, "beta"),
                               _dev(end, "end", torch.int32), float(K_IC),
                               _dev(grow, "grow", torch.int32), _dev(nx, "nx"), _dev(ny, "ny"),
                               _dev(na, "na"), _dev(nb, "nb"), _dev(ne, "ne", torch.int32),
                               _stream_ptr(stream)))
    return grow, nx, ny, na, nb, ne


def shard_owner(c_start: np.ndarray, c_count: np.ndarray, rank_el_lo: np.ndarray) -> np.ndarray:
    """Host-only ddm_shard_owner: the rank on which each cell is complete, or -1
    (straddling cell)."""
    st = np.ascontiguousarray(c_start, dtype=np.int32)
    ct = np.ascontiguousarray(c_count, dtype=np.int32)
    lo = np.ascontiguousarray(rank_el_lo, dtype=np.int64)
    out = np.empty(st.size, dtype=np.int32)
    rc = L.ddm_shard_owner(st.ctypes.data_as(C.POINTER(C.c_int)), ct.ctypes.data_as(C.POINTER(C.c_int)),
                           int(st.size), lo.ctypes.data_as(C.POINTER(C.c_int64)), int(lo.size - 1),
                           out.ctypes.data_as(C.POINTER(C.c_int)))
    if rc != L.OK:
        raise DDMError(rc, "ddm_shard_owner")
    return out


def split_costs(prefix_excl: np.ndarray, total: int, world: int) -> np.ndarray:
    """Host-only leaf partition (ddm_split_costs); no GPU needed."""
    pre = np.ascontiguousarray(prefix_excl, dtype=np.int64)
    out = np.empty(world + 1, dtype=np.int32)
    rc = L.ddm_split_costs(pre.ctypes.data_as(C.POINTER(C.c_int64)), int(total), int(pre.size),
                           int(world), out.ctypes.data_as(C.POINTER(C.c_int)))
    if rc != L.OK:
        raise DDMError(rc, "ddm_split_costs")
    return out
