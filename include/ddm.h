/*
 * ddm.h — C-ABI of the B200-native FMM displacement-discontinuity library
 * (libddm.so).  Plain pointers and sizes only; no torch or CUDA types.
 *
 * The operation this library accelerates is the matrix–vector product of the
 * constant-element displacement discontinuity method (DDM), PAPER.md
 * Eq.(final_sigs)–Eq.(final_pp): for N constant elements,
 *
 *     y_beta = sum_lambda A^{beta lambda} D^lambda ,
 *
 * "nine matrix-vector multiplications ... at each iteration" of GMRES and for
 * "any extra time step", applied matrix-free through a fast
 * multipole method (§3) at both of the paper's modification sites:
 * the GMRES operator apply and the time-marching history sum (P:469-473,
 * P:922-931).
 *
 * Conventions:
 *   - Element i: centre (xc[i], yc[i]), half-length a[i] > 0, direction angle
 *     beta[i] (tangent s = (cos, sin), normal n = (-sin, cos)).
 *   - DOF layout element-major interleaved: D[ncomp*i + c], c = 0 shear D_s,
 *     1 normal D_n (opening positive), 2 fluid source D_q (poroelastic only).
 *     Rows: (sigma_s, sigma_n[, p]) at element i's centre, compression
 *     positive.  ncomp = 2 elastic, 3 poroelastic.
 *   - Collocation at element centres.
 *   - All floating point is IEEE fp64.
 *
 * Ownership: every array argument is caller-owned and only read (const) or
 * written (non-const); the library keeps no pointer to caller memory after a
 * call returns.  Pointers marked [device] must be CUDA device memory on the
 * context's device; [host] must be host memory.  `stream` is a cudaStream_t
 * passed as void* (NULL = legacy default stream); every call is ordered on
 * it, and calls that return data to the host synchronise it.
 *
 * Errors: every int-returning call returns a ddm_status; on failure a
 * message is available from ddm_last_error(ctx) until the next call on that
 * context.  No call aborts the process.
 */
#ifndef DDM_H_
#define DDM_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DDM_OK = 0,
  DDM_ERR_ARG = 1,     /* invalid argument / dimension / material mismatch   */
  DDM_ERR_CUDA = 2,    /* CUDA runtime error                                  */
  DDM_ERR_NOCONV = 3,  /* GMRES did not converge: x = best iterate            */
  DDM_ERR_NCCL = 4,    /* NCCL error                                          */
  DDM_ERR_GEOM = 5,    /* non-finite coordinates or coincident points at the
                          depth cap                                           */
  DDM_ERR_OOM = 6      /* device allocation failed                            */
} ddm_status;

enum { DDM_FMM = 0, DDM_DIRECT = 1,
       DDM_HIST_PERLAG = 2, /* ddm_history_apply only: one FMM matvec per lag (the paper's scheme) */
       DDM_GMRES_NO_PRECOND = 8, /* ddm_gmres_solve only, OR-ed into mode: plain GMRES */
       DDM_GMRES_PC_POINT = 32,  /* ddm_gmres_solve only, OR-ed into mode: point-block
                                    Jacobi (element self blocks) instead of leaf blocks */
       DDM_BBFMM = 16 /* ddm_matvec / ddm_gmres_solve, elastic: the paper's Chebyshev
                         (bbFMM) far field with n nodes per dimension, mode =
                         DDM_BBFMM_MODE(n), 2 <= n <= 8 */ };
#define DDM_BBFMM_MODE(n) (DDM_BBFMM | ((n) << 8))

/* Material (Table rock_prop).  kind 0 = elastic (only G,
 * nu used), 1 = fully coupled poroelastic.  kappa = k / mu (m^2 / (Pa s)). */
typedef struct {
  int kind;
  double G, nu, nu_u, alpha, kappa;
} ddm_material;

typedef struct ddm_ctx_s* ddm_ctx_t;
typedef struct ddm_tree_s* ddm_tree_t;

/* ---------------------------------------------------------------- context
 * ddm_ctx_create: bind to CUDA `device`.  nccl_uid: NULL for a single GPU,
 * else the 128-byte ncclUniqueId that rank 0 created (ddm_nccl_unique_id) and
 * the caller broadcast (torch.distributed is used only for that broadcast).
 * rank / world: this process's place in the one-process-per-GPU job. */
int ddm_ctx_create(int device, const void* nccl_uid, int rank, int world, ddm_ctx_t* out);
void ddm_ctx_destroy(ddm_ctx_t ctx);
const char* ddm_last_error(ddm_ctx_t ctx);
/* Writes a fresh ncclUniqueId (128 bytes) into uid_out [host]. */
int ddm_nccl_unique_id(void* uid_out);
/* Library version string, e.g. "ddm-b200 0.1 sm_100a". */
const char* ddm_version(void);

/* ---------------------------------------------------------------- tree
 * ddm_build_tree — hierarchical tree decomposition: Morton keys
 * (a1), stable LSD radix sort (a2), cells (a3) and U/V interaction lists (a4)
 * of DESIGN.md §4.  xc, yc, half_len, beta [device], n elements, user order.
 * leaf_size: "prescribed number" of P:585 (>= 1).  order_p: number of
 * complex coefficients per expansion series (2 <= p <= 40).
 * min_leaf_side: depth cap, no cell is split below this side (0 = none).
 * The tree is built once per geometry and reused.
 * Errors: n < 1, leaf_size < 1, bad p -> DDM_ERR_ARG; non-finite coordinates
 * or more than leaf_size coincident centres at depth 30 -> DDM_ERR_GEOM.
 * The tree owns its device buffers until ddm_tree_free.  Multi-GPU: every
 * rank passes the full geometry and builds the same tree; each rank then owns
 * a contiguous range of Morton-ordered leaves (ddm_tree_partition). */
int ddm_build_tree(ddm_ctx_t ctx, const double* xc, const double* yc, const double* half_len,
                   const double* beta, int64_t n, int leaf_size, int order_p,
                   double min_leaf_side, void* stream, ddm_tree_t* out);
/* Releases every device buffer, captured graph and pinned host buffer of the
 * tree.  The tree may still be in use on any stream of the caller's, so the
 * call waits for the device to go idle first (cudaFree would synchronise
 * anyway); NULL is a no-op. */
void ddm_tree_free(ddm_tree_t tree);

/* Sizes of the tree's arrays, written into counts[DDM_TREE_NCOUNTS] [host].
 * X = X-list entries (P2L source leaves), X_MIN = the target
 * leaf size from which X lists are built (env DDM_X_MIN at build time,
 * default 0 = off: measured slower on config 5),
 * UXRANGES = merged ranges of U minus X, and
 * NEAR_PAIRS_P2P = the (target, source) pairs the elastic series-FMM near
 * field evaluates (NEAR_PAIRS minus the X pairs). */
enum {
  DDM_TC_N = 0, DDM_TC_CELLS, DDM_TC_LEAVES, DDM_TC_LEVELS, DDM_TC_V, DDM_TC_URANGES,
  DDM_TC_NEAR_PAIRS, DDM_TC_P2P_ITEMS, DDM_TC_OWNED_LO, DDM_TC_OWNED_HI, DDM_TC_P,
  DDM_TC_W, DDM_TC_W_MIN, DDM_TC_X, DDM_TC_X_MIN, DDM_TC_UXRANGES, DDM_TC_NEAR_PAIRS_P2P,
  DDM_TREE_NCOUNTS = 20
};
int ddm_tree_counts(ddm_tree_t tree, int64_t* counts);

/* Multi-rank matvec emulated on ONE device (tests of the sharded path,
 * DESIGN.md §6): trees[r] [host array of handles] is one geometry built on
 * this context and partitioned (ddm_tree_partition) as rank r of `world`.
 * Runs the elastic FMM matvec exactly as `world` ranks would (each rank's
 * near field, P2M of its leaves and M2M of its complete cells, the multipole
 * all-gather, the straddling cells' M2M, the downward pass and assembly of
 * its owned rows), rank by rank on `stream`, with device copies in place of
 * the NCCL all-gathers.  D, y: device [n][2], user order.  Elastic only
 * (DDM_ERR_ARG otherwise).  The result equals ddm_matvec on the unpartitioned
 * tree bitwise: every row is summed in the same order. */
int ddm_matvec_sim(ddm_ctx_t ctx, const ddm_tree_t* trees, int world, const ddm_material* mat,
                   const double* D, double* y, void* stream);

/* Timing of the last ddm_build_tree of `tree` (keys, sort, cells,
 * interaction lists; built once per geometry), written into
 * ms[DDM_TB_N] [host], milliseconds: stage spans from CUDA events on the build
 * stream (host gaps included) and the host wall time of the whole call
 * (operators and partition included).  Always available; no profiling mode. */
enum { DDM_TB_KEYS = 0, DDM_TB_SORT, DDM_TB_CELLS, DDM_TB_LISTS, DDM_TB_SCHED, DDM_TB_TOTAL,
       DDM_TB_N };
int ddm_tree_build_times(ddm_tree_t tree, double* ms);

/* Copy one exported array into dst [host] (capacity in bytes).  Arrays:
 *   KEYS    u64[n]   Morton key of each element, user order
 *   PERM    i32[n]   sorted position -> user index
 *   ROOT    f64[3]   x_min, y_min, W
 *   LEVEL   i32[c], IX i32[c], IY i32[c], START i32[c], COUNT i32[c],
 *   PARENT  i32[c], FIRST_CHILD i32[c], NCHILD i32[c], LEAF i32[c]
 *   V_OFF   i32[c+1], V_IDX i32[nv]            (CSR, per target cell)
 *   LEAVES  i32[nl]  cell index of each leaf (canonical order)
 *   U_OFF   i32[nl+1], U_LO i32[nu], U_HI i32[nu]   (CSR of source element
 *           ranges [lo, hi) in sorted order, per leaf; sorted and merged)
 *   W_OFF   i32[nl+1], W_IDX i32[nw]   (CSR of M2P source cells per leaf,
 *           ascending, the W split of R5: cells deeper than the
 *           leaf, not touching it, with >= w_min elements; env DDM_W_MIN at
 *           build time, default 24, 0 = no W lists)
 *   X_OFF   i32[nl+1], X_IDX i32[nx]   (CSR of P2L source leaves per target
 *           leaf, ascending element start, the dual of W:
 *           leaves of U coarser than the target leaf and not touching it,
 *           for target leaves of >= x_min elements)
 *   UX_OFF  i32[nl+1], UX_LO i32[nux], UX_HI i32[nux]   (U minus X, as U) */
enum {
  DDM_EX_KEYS = 0, DDM_EX_PERM, DDM_EX_ROOT, DDM_EX_LEVEL, DDM_EX_IX, DDM_EX_IY,
  DDM_EX_START, DDM_EX_COUNT, DDM_EX_PARENT, DDM_EX_FIRST_CHILD, DDM_EX_NCHILD,
  DDM_EX_LEAF, DDM_EX_V_OFF, DDM_EX_V_IDX, DDM_EX_LEAVES, DDM_EX_U_OFF, DDM_EX_U_LO,
  DDM_EX_U_HI, DDM_EX_W_OFF, DDM_EX_W_IDX, DDM_EX_X_OFF, DDM_EX_X_IDX, DDM_EX_UX_OFF,
  DDM_EX_UX_LO, DDM_EX_UX_HI
};
int ddm_tree_export(ddm_tree_t tree, int what, void* dst, int64_t capacity_bytes);

/* Partition the Morton-ordered leaves into `world` contiguous ranges of
 * near-equal estimated cost (P2P pairs + M2L work) and keep rank's range.
 * Called automatically by ddm_build_tree with the context's rank/world. */
int ddm_tree_partition(ddm_tree_t tree, int rank, int world);

/* Host-only helper (no GPU needed) of the sharded upward pass:
 * owner[c] = the rank r whose sorted-element range [rank_el_lo[r],
 * rank_el_lo[r+1]) contains cell c's whole range [c_start[c], c_start[c] +
 * c_count[c]) (a COMPLETE cell: r computes its multipole from its own
 * elements), or -1 for a straddling cell (its range crosses a rank boundary;
 * completed on every rank from its children after the multipole
 * all-gather).  All arrays host memory; rank_el_lo has world+1 entries. */
int ddm_shard_owner(const int* c_start, const int* c_count, int ncells,
                    const int64_t* rank_el_lo, int world, int* owner);

/* Host-only helper (no GPU needed): split leaves with exclusive cost prefix
 * prefix_excl[nleaves] (total = sum of costs) into `world` contiguous ranges:
 * split[r] = first leaf of rank r, split[world] = nleaves.  Rank r gets the
 * leaves whose prefix lies in [r total / world, (r+1) total / world). */
int ddm_split_costs(const int64_t* prefix_excl, int64_t total, int nleaves, int world,
                    int* split);

/* ---------------------------------------------------------------- matvec
 * y = A(elapsed) D (Eq.(final_sigs)-(final_pp) left-hand side).
 * D, y [device], [n][ncomp] user order.  mode DDM_FMM: the FMM of DESIGN.md
 * §4 (P2M, M2M, M2L, L2L, L2P + exact near-field P2P).
 * mode DDM_DIRECT: exact all-pairs evaluation (no expansions).
 * mode DDM_BBFMM_MODE(n) (elastic only): the same tree, lists and exact near
 * field, far field by the paper's black-box FMM -- Chebyshev interpolation
 * with n x n nodes per cell (S_n), node weights (Eq.(p2l),
 * Eq.(m2m)), kernel at node pairs (Eq.(m2l)), interpolation down the tree
 * (Eq.(l2l)) and at the targets; DESIGN.md §4.9.  Accuracy is the
 * interpolation's (n = 3: ~1e-4, n = 6: ~1e-6 relative), not the series'.
 * Errors: n outside [2, 8] or a poroelastic material -> DDM_ERR_ARG.
 * elapsed is the
 * time since the constant source was switched on (poroelastic; ignored when
 * elastic).  Multi-GPU: D and y are full-length on every rank; y is complete
 * on every rank on return (owned slices exchanged with NCCL all-gather).
 * Errors: material/kind mismatch -> DDM_ERR_ARG. */
int ddm_matvec(ddm_ctx_t ctx, ddm_tree_t tree, const ddm_material* mat, double elapsed,
               const double* D, double* y, int mode, void* stream);

/* r = sum_{m=1}^{h} A^{(m)} D^{h-m}, A^{(m)} = K((m+1) dt) - K(m dt)
 * (history double sum of Eq.(final_sigs)-(final_pp); P:922-929;
 * reading R10).  D_hist [device] [h][n][3] user order (D^0 .. D^{h-1}, the
 * caller's storage, only read); r [device] [n][3] user order, overwritten.
 * h = 0 or elastic -> r = 0.  Written as r = sum_{j=1}^{h+1} K(j dt) E_j,
 * E_j = D^{h+1-j} - D^{h-j}.  mode DDM_FMM: fast form -- one
 * far-field pass of the tau-linear far weights on sum_{k<h} D^k plus one
 * multi-lag near-field launch; needs a tree built with min_leaf_side >=
 * sqrt(160 c (h+1) dt) + 2 max(a) (else DDM_ERR_ARG).  DDM_HIST_PERLAG: h+1
 * FMM matvecs (the paper's one-FMM-per-previous-step scheme).
 * DDM_DIRECT: h+1 exact all-pairs matvecs.  Multi-GPU: r complete on every
 * rank. */
int ddm_history_apply(ddm_ctx_t ctx, ddm_tree_t tree, const ddm_material* mat, double dt,
                      int h, const double* D_hist, double* r, int mode, void* stream);

/* Right-hand side of step h of the time marching ("subtracting
 * the effect of all previous time steps"): rhs = b - sum_{m=1}^{h} A^{(m)} D^{h-m}
 * (ddm_history_apply with the same mode and errors).  b, rhs [device] [n][3]
 * user order (may alias). */
int ddm_history_rhs(ddm_ctx_t ctx, ddm_tree_t tree, const ddm_material* mat, double dt, int h,
                    const double* D_hist, const double* b, double* rhs, int mode, void* stream);

/* GMRES initial guess for step h of the time marching (not part of the
 * paper's method, which solves every step from its own start; DESIGN.md §4.7c:
 * it only changes the iteration count, every step is still solved to the
 * same true residual).  x = polynomial extrapolation in time of the previous
 * solutions, sum_{j=1}^{q+1} (-1)^{j+1} C(q+1, j) D^{h-j} summed left to right:
 * order 5: 6 D^{h-1} - 15 D^{h-2} + 20 D^{h-3} - 15 D^{h-4} + 6 D^{h-5} - D^{h-6};
 * 4: 5 D^{h-1} - 10 D^{h-2} + 10 D^{h-3} - 5 D^{h-4} + D^{h-5};
 * 3: 4 D^{h-1} - 6 D^{h-2} + 4 D^{h-3} - D^{h-4}; 2: 3 (D^{h-1} - D^{h-2}) + D^{h-3};
 * 1: 2 D^{h-1} - D^{h-2}; 0: D^{h-1}; the order is lowered to h - 1 while
 * fewer steps exist; h = 0 -> x = 0.  D_hist [device] [h][len] (D^0 .. D^{h-1},
 * only read), x [device] [len], written.  Errors: h < 0, len < 0, order < 0
 * or > 5, NULL x (or NULL D_hist with h > 0) -> DDM_ERR_ARG. */
int ddm_march_guess(ddm_ctx_t ctx, int h, const double* D_hist, int64_t len, int order, double* x,
                    void* stream);

/* GMRES (reading R11): solve A(dt) x = b with classical
 * Gram-Schmidt Arnoldi (second pass when the first cancels more than half of
 * ||w||^2), Givens rotations, restart `restart`, relative tolerance tol on
 * ||b - A x|| / ||b|| (the true residual: right preconditioning; a cycle
 * whose estimate reaches tol is continued, not restarted, until the true
 * residual does).  Preconditioner: by default leaf-block
 * Jacobi -- the exact dense blocks of chunks of <= 32 consecutive elements
 * of one leaf (the strongest couplings: neighbours on the same fracture),
 * inverted once per material / dt; DDM_GMRES_PC_POINT OR-ed into mode: the
 * element self blocks (2x2 elastic / 3x3 poroelastic); DDM_GMRES_NO_PRECOND:
 * none.  The operator mode is DDM_FMM, DDM_DIRECT or DDM_BBFMM_MODE(n).
 * b, x [device] [n][ncomp]; x holds the initial guess
 * on entry and the solution on return.  iters, rel_resid [host] outputs
 * (rel_resid = explicit true residual at exit).  b = 0 -> x = 0, iters = 0.
 * Returns DDM_ERR_NOCONV with x = last iterate if max_iter is reached. */
/* y = M^-1 x, the GMRES preconditioner on its own: kind 1
 * point-block Jacobi (inverse element self blocks), kind 2 leaf-block Jacobi
 * (inverse dense blocks of <= 32 consecutive elements of one leaf; chunks as
 * documented at ddm_gmres_solve).  x, y [device] [n][ncomp] user order.
 * Errors: kind not 1/2, poroelastic with dt <= 0 -> DDM_ERR_ARG. */
int ddm_precond_apply(ddm_ctx_t ctx, ddm_tree_t tree, const ddm_material* mat, double dt,
                      const double* x, double* y, int kind, void* stream);

int ddm_gmres_solve(ddm_ctx_t ctx, ddm_tree_t tree, const ddm_material* mat, double dt,
                    const double* b, double* x, double tol, int restart, int max_iter,
                    int mode, int* iters, double* rel_resid, void* stream);

/* Right-hand side of the first step: far-field stresses (sH along
 * x, sh along y, compression positive) resolved on each face, plus the
 * hydraulic load: b_s = (sH - sh) sin b cos b; b_n = p_f - sigma_n^ff
 * (net = 0) or p_f (net = 1); b_p = p_f_pore (poroelastic).  beta [device],
 * b [device] [n][ncomp]. */
int ddm_farfield_rhs(ddm_ctx_t ctx, const double* beta, int64_t n, int ncomp, double p_f,
                     double sH, double sh, int net, double b_p, double* b, void* stream);

/* Stress intensity factors, Olson's formula Eq.(SIF):
 * K = 0.806 E / (4 (1 - nu^2)) sqrt(pi / (2 a)) D.  w_tip (= D_n), ds_tip,
 * a_tip, KI, KII [device] length ntips. */
int ddm_sif(ddm_ctx_t ctx, const double* w_tip, const double* ds_tip, const double* a_tip,
            int ntips, double E, double nu, double* KI, double* KII, void* stream);

/* Fracture propagation step (Fig. 8 branch: "a fracture
 * propagation criterion may be used ... an element will be added to the
 * model if propagation happens, and in that case the quad-tree needs to be
 * constructed again").  The paper names no criterion; reading
 * R23: maximum tangential stress (Erdogan-Sih) in each tip's
 * outward frame, kink angle theta = 2 atan((K_I - sqrt(K_I^2 + 8 K_II^2)) /
 * (4 K_II)) (0 when K_II = 0), K_eq = cos(theta/2) (K_I cos^2(theta/2) -
 * 3/2 K_II sin theta); a tip grows when K_I > 0 and K_eq >= K_IC, by one
 * element of the tip element's length along phi = outward angle + theta.
 * Per tip i (all arrays [device], length ntips): KI, KII (ddm_sif); the tip
 * element's centre (x, y), half-length a, angle beta in [0, pi) and end
 * (1: its (x, y) + a e^{i beta} endpoint is the tip, 0: the - endpoint).
 * Outputs: grow[i] (0/1) and, where grow[i] = 1, the new element (new_x,
 * new_y, new_a, new_beta in [0, pi)) and its outward end new_end.  The caller
 * appends the new elements and rebuilds the tree (ddm_build_tree).  Errors:
 * DDM_ERR_ARG for NULL arrays with ntips > 0 or K_IC < 0. */
int ddm_tip_growth(ddm_ctx_t ctx, int ntips, const double* KI, const double* KII,
                   const double* x, const double* y, const double* a, const double* beta,
                   const int* end, double K_IC, int* grow, double* new_x, double* new_y,
                   double* new_a, double* new_beta, int* new_end, void* stream);

/* Per-stage timings of the last ddm_matvec on this tree (CUDA events, ms),
 * written into ms[DDM_NSTAGES] [host] when profiling is enabled
 * (ddm_set_profiling).  Stages: prep, p2m, m2m, m2l, l2l, p2p, finalize (near +
 * far sum and scatter), exchange, l2p, p2l (X lists).  enable = 0: off; 1: events on the normal schedule (the near
 * field runs concurrently with the far-field chain, so stage times overlap);
 * 2: events + serial schedule (every stage on the caller's stream, one after
 * another: each stage time is that stage's kernels alone, for rooflines). */
enum { DDM_ST_PREP = 0, DDM_ST_P2M, DDM_ST_M2M, DDM_ST_M2L, DDM_ST_L2L, DDM_ST_P2P,
       DDM_ST_FINAL, DDM_ST_COMM, DDM_ST_L2P, DDM_ST_P2L, DDM_NSTAGES };
int ddm_set_profiling(ddm_ctx_t ctx, int enable);
int ddm_stage_times(ddm_ctx_t ctx, double* ms);

/* Measured fp64 FMA throughput of this GPU (TFLOP/s, FMA = 2 flop), from a
 * DFMA-chain kernel on all SMs, best of 5 (the roofline denominator for the
 * fp64-ALU-bound kernels).  tflops [host]. */
int ddm_probe_fp64(ddm_ctx_t ctx, double* tflops, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* DDM_H_ */
