// FMM matvec driver for the elastic constant-DD kernel and the
// host-side construction of the (scale-free) translation operators.
//
// PAPER.md §3.2: upward pass (P2M "P2L", M2M), downward pass (M2L
// over interaction lists, L2L), final L2P + P2P for self and neighbour cells.
// The paper's Chebyshev interpolation (bbFMM) is replaced by complex-variable
// (Kolosov–Muskhelishvili) expansions of the constant-element influence.
#include <cstring>
#include <algorithm>
#include <cmath>
#include <vector>

#include "kcommon.cuh"

namespace ddm {
namespace {

double binom(int n, int k) {
  if (k < 0 || k > n) return 0.0;
  double r = 1.0;
  for (int i = 1; i <= k; ++i) r = r * (n - k + i) / i;
  return r;
}

}  // namespace

// Per-tree FMM workspaces (expansions, source records, partials, sorted
// outputs) and the near-field source stream; idempotent.
int fmm_workspace(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) {
  int rc;
  if (!t->mpole) {
    if ((rc = talloc(ctx, &t->mpole, (size_t)t->ncells * 2 * t->p, s))) return rc;
    if ((rc = talloc(ctx, &t->local, (size_t)t->ncells * 2 * t->p, s))) return rc;
    if ((rc = talloc(ctx, &t->src, (size_t)t->n * kSrcStride, s))) return rc;
    if ((rc = talloc(ctx, &t->part, (size_t)t->nitems * kTgtGroup * 2, s))) return rc;  // <= 4 doubles/slot
    if ((rc = talloc(ctx, &t->d_sorted, (size_t)t->n * 3, s))) return rc;
    if ((rc = talloc(ctx, &t->y_sorted, (size_t)t->n * 3, s))) return rc;
    if ((rc = talloc(ctx, &t->y_far, (size_t)t->n * 3, s))) return rc;
    if ((rc = talloc(ctx, &t->y_near, (size_t)t->n * 2, s))) return rc;
  }
  if ((rc = build_source_stream(ctx, t, s))) return rc;
  return l2p_prepare(ctx, t, s);
}


// Translation operators (host, fp64), uploaded once per tree.  Every
// translation of DESIGN.md §4 factors as  post-scale x (real Pascal matrix) x
// pre-scale  (the binomial expansions of Eq.(m2m), Eq.(m2l), Eq.(l2l) with the
// offset powers pulled out of the sums):
//   M2M  alpha^P_{m+1} = eps^{m+1} sum_n C(m, n) (2 eps)^{-(n+1)} alpha^q_{n+1}
//   M2L  lambda_m      = (-w)^m    sum_n C(m+n, n) w^{n+1} alpha_{n+1}
//   L2L  l^c_k         = (2 eps)^{-k} sum_m C(m, k) eps^m lambda^P_m
// eps = (z_child - z_parent)/s_parent (4 quadrants), w = 1/delta with
// delta = (z_target - z_source)/s = -(dx + i dy) for the 49 offset classes
// o = (dy+3)*7 + (dx+3) (classes with max(|dx|,|dy|) < 2 are unused).
int fmm_init_operators(ddm_tree_s* t, cudaStream_t s) {
  ddm_ctx_s* ctx = t->ctx;
  const int p = t->p;
  typedef std::vector<double2> V;
  std::vector<double> pas((size_t)p * p), pasT((size_t)p * p), pm2l((size_t)(p + 1) * p);
  for (int m = 0; m < p; ++m)
    for (int k = 0; k < p; ++k) {
      pas[(size_t)m * p + k] = binom(m, k);
      pasT[(size_t)k * p + m] = binom(m, k);
    }
  for (int n = 0; n <= p; ++n)
    for (int m = 0; m < p; ++m) pm2l[(size_t)n * p + m] = binom(m + n, n);
  auto cmulh = [](double2 a, double2 b) {
    return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
  };
  const int pw = p + 2;
  V eps((size_t)4 * pw), e2i((size_t)4 * pw), w((size_t)kNOffsets * pw, make_double2(0.0, 0.0));
  for (int q = 0; q < 4; ++q) {
    const double2 e = make_double2(0.5 * ((q & 1) - 0.5), 0.5 * ((q >> 1) - 0.5));
    const double n2 = 4.0 * (e.x * e.x + e.y * e.y);
    const double2 ie = make_double2(2.0 * e.x / n2, -2.0 * e.y / n2);   // 1/(2 eps)
    double2 a = make_double2(1.0, 0.0), b = a;
    for (int k = 0; k < pw; ++k) {
      eps[(size_t)q * pw + k] = a;
      e2i[(size_t)q * pw + k] = b;
      a = cmulh(a, e);
      b = cmulh(b, ie);
    }
  }
  for (int o = 0; o < kNOffsets; ++o) {
    const int dx = o % 7 - 3, dy = o / 7 - 3;
    if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
    const double r2 = (double)dx * dx + (double)dy * dy;
    const double2 wo = make_double2(-dx / r2, dy / r2);   // 1/delta = conj(delta)/|delta|^2
    double2 a = make_double2(1.0, 0.0);
    for (int k = 0; k < pw; ++k) {
      w[(size_t)o * pw + k] = a;
      a = cmulh(a, wo);
    }
  }
  int rc;
  if ((rc = talloc(ctx, &t->op_pas, pas.size(), s)) || (rc = talloc(ctx, &t->op_pasT, pasT.size(), s)) ||
      (rc = talloc(ctx, &t->op_pm2l, pm2l.size(), s)) || (rc = talloc(ctx, &t->op_w, w.size(), s)) ||
      (rc = talloc(ctx, &t->op_eps, eps.size(), s)) || (rc = talloc(ctx, &t->op_e2i, e2i.size(), s)))
    return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_pas, pas.data(), pas.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_pasT, pasT.data(), pasT.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_pm2l, pm2l.data(), pm2l.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_w, w.data(), w.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_eps, eps.data(), eps.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_e2i, e2i.data(), e2i.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  return DDM_OK;
}

// Matvec y = A(elapsed) D.  D: [n][ncomp], user order
// (d_sorted = false) or sorted order, full length on every rank; ncomp = 2
// elastic, 3 poroelastic.  Writes the owned rows into y_user (user order)
// and/or y_sorted (sorted order).
static int fmm_matvec_launch(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat,
                             double elapsed, const double* D, bool d_sorted, double* y_user,
                             double* y_sorted, int mode, cudaStream_t s);

void drop_graphs(ddm_tree_s* t) {
  if (t->gm_exec) cudaGraphExecDestroy(t->gm_exec);
  t->gm_exec = nullptr;
  for (auto& g : t->graphs) {
    if (g.exec) cudaGraphExecDestroy(g.exec);
    g.exec = nullptr;
    g.key = MatvecKey();
  }
  for (auto& k : t->seen_keys) k = MatvecKey();
  t->graph_next = t->seen_next = 0;
}

// CUDA-graph replay of the matvec launch sequence (23 launches for config 5,
// fork/join across the two streams captured as graph edges): a call whose
// arguments (pointers, material, elapsed time, mode, stream) repeat the
// previous call's is captured once and then replayed, so repeated matvecs
// (GMRES operator, benchmark steps) pay one graph launch instead of the
// per-kernel launch overhead.  Profiling (per-stage events) bypasses graphs;
// DDM_NO_GRAPH=1 disables them.
int fmm_matvec(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double elapsed,
               const double* D, bool d_sorted, double* y_user, double* y_sorted, int mode,
               cudaStream_t s) {
  int rc = fmm_workspace(ctx, t, s);
  if (rc) return rc;
  // poroelastic near-field blocks: cached for repeated matvecs at one elapsed
  // time (GMRES), outside any capture
  if (mat->kind == 1 && mode == DDM_FMM && elapsed > 0)
    if ((rc = poro_near_cache_update(ctx, t, poro_params(mat, elapsed), s))) return rc;
  // bbFMM node arrays sized for this order, also outside any capture (a
  // change of order reallocates them and drops the graphs that used them)
  if ((mode & DDM_BBFMM) && mat->kind == 0)
    if ((rc = bb_prepare(ctx, t, (mode >> 8) & 0xff))) return rc;
  static const bool no_graph = [] {
    const char* e = getenv("DDM_NO_GRAPH");
    return e && e[0] == '1';
  }();
  // several ranks: the sharded upward pass all-gathers multipoles inside the
  // far chain (NCCL), launched directly rather than captured
  // inside a capture (the GMRES step graph) the launches become its nodes
  cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &cst) != cudaSuccess) {
    cudaGetLastError();
    cst = cudaStreamCaptureStatusNone;
  }
  if (ctx->profiling || no_graph || !ctx->s_cap || ctx->world > 1 ||
      cst != cudaStreamCaptureStatusNone)
    return fmm_matvec_launch(ctx, t, mat, elapsed, D, d_sorted, y_user, y_sorted, mode, s);
  MatvecKey key;
  key.D = D;
  key.y_user = y_user;
  key.y_sorted = y_sorted;
  key.s = s;
  key.mode = mode;
  key.d_sorted = d_sorted;
  key.mat = *mat;
  key.elapsed = mat->kind == 1 ? elapsed : 0.0;
  key.serial = ctx->serial;
  for (auto& g : t->graphs)
    if (g.exec && g.key == key) {
      DDM_CUDA(ctx, cudaGraphLaunch(g.exec, s));
      return DDM_OK;
    }
  // capture on the second use of the same arguments among the last four
  // argument sets (alternating buffers, e.g. a pipelined caller, repeat too)
  bool seen = false;
  for (const auto& k : t->seen_keys) seen = seen || (k == key);
  if (!seen) {
    t->seen_keys[t->seen_next] = key;
    t->seen_next = (t->seen_next + 1) % 4;
    return fmm_matvec_launch(ctx, t, mat, elapsed, D, d_sorted, y_user, y_sorted, mode, s);
  }
  // captured on the library's own stream (the caller's may be the legacy
  // default stream, which cannot be captured); replayed on the caller's
  cudaGraph_t graph = nullptr;
  const cudaStream_t sc = ctx->s_cap;
  DDM_CUDA(ctx, cudaStreamBeginCapture(sc, cudaStreamCaptureModeThreadLocal));
  rc = fmm_matvec_launch(ctx, t, mat, elapsed, D, d_sorted, y_user, y_sorted, mode, sc);
  const cudaError_t ce = cudaStreamEndCapture(sc, &graph);
  if (rc) {
    if (graph) cudaGraphDestroy(graph);
    return rc;
  }
  if (ce != cudaSuccess) return cuda_error(ctx, ce, "cudaStreamEndCapture");
  cudaGraphExec_t exec = nullptr;
  // honour the stream priorities captured into the nodes (near field low, far chain high)
  const cudaError_t ie =
      cudaGraphInstantiateWithFlags(&exec, graph, cudaGraphInstantiateFlagUseNodePriority);
  cudaGraphDestroy(graph);
  if (ie != cudaSuccess) return cuda_error(ctx, ie, "cudaGraphInstantiate");
  // keep a few graphs (round robin)
  auto& slot = t->graphs[t->graph_next];
  t->graph_next = (t->graph_next + 1) % (int)t->graphs.size();
  if (slot.exec) cudaGraphExecDestroy(slot.exec);
  slot.exec = exec;
  slot.key = key;
  DDM_CUDA(ctx, cudaGraphLaunch(exec, s));
  return DDM_OK;
}

static int fmm_matvec_launch(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat,
                             double elapsed, const double* D, bool d_sorted, double* y_user,
                             double* y_sorted, int mode, cudaStream_t s) {
  int rc = DDM_OK;
  const bool poro = mat->kind == 1;
  const int ncomp = poro ? 3 : 2;
  const double gc = mat->G / (4.0 * M_PI * (1.0 - mat->nu));
  const int64_t lo = t->own_el_lo, hi = t->own_el_hi;
  const int* perm_in = d_sorted ? nullptr : t->perm;
  PoroParams PP;
  PoroFar pf;
  if (poro) {
    if (!(elapsed > 0)) return set_error(ctx, DDM_ERR_ARG, "poroelastic matvec needs elapsed > 0");
    PP = poro_params(mat, elapsed);
    pf = poro_far(PP);
    if (mode == DDM_FMM && t->nlevels > 2) {
      // the far field is the r >> sqrt(c tau) form: every V pair must be
      // separated by more than R_c = sqrt(160 c tau) (u > 40)
      const double smin = std::ldexp(t->W, -(t->nlevels - 1));
      const double sep = smin - 2.0 * t->a_max;
      if (sep <= 0 || sep * sep / (4.0 * PP.ct) <= 40.0)
        return set_error(ctx, DDM_ERR_ARG,
                         "tree too fine for the poroelastic far field at this elapsed time: build "
                         "it with min_leaf_side >= sqrt(160 c tau) + 2 max(a)");
    }
  }

  // DDM_SHARD_NOEXCHANGE=1 (scripts/rank_timing.py only): one process times
  // a rank's sharded work on a partitioned tree WITHOUT the multipole
  // exchange -- the far field is then incomplete, the result invalid
  static const bool noexch = [] {
    const char* e = getenv("DDM_SHARD_NOEXCHANGE");
    return e && e[0] == '1';
  }();

  // Chebyshev far field (f2, bbfmm.cu): mode DDM_BBFMM | n << 8, elastic
  const bool bb = (mode & DDM_BBFMM) != 0;
  const int bb_n = (mode >> 8) & 0xff;
  if (bb) {
    if (poro) return set_error(ctx, DDM_ERR_ARG, "the bbFMM far field is elastic only");
    if ((rc = bb_prepare(ctx, t, bb_n))) return rc;
  }

  // The series far field reads D itself (P2M through perm), so it does not
  // wait for the near field's source records: fork first, prep on the near
  // stream (the far chain starts at once; it is the critical path on small
  // trees).  DDM_EARLY_FAR=0: prep before the fork (P2M reads D sorted).
  static const bool early_env = [] {
    const char* e = getenv("DDM_EARLY_FAR");
    return !(e && e[0] == '0');
  }();
  const bool early = early_env && !bb && mode != DDM_DIRECT;
  cudaStream_t sf = ctx->serial ? s : ctx->s_hi, sn = ctx->serial ? s : ctx->s_lo;
  if (early) {
    DDM_CUDA(ctx, cudaEventRecord(ctx->ev_fork, s));
    DDM_CUDA(ctx, cudaStreamWaitEvent(sf, ctx->ev_fork, 0));
    DDM_CUDA(ctx, cudaStreamWaitEvent(sn, ctx->ev_fork, 0));
  }
  cudaStream_t sp = early ? sn : s;
  stage_begin(ctx, DDM_ST_PREP, sp);
  // elastic: the direct mode reads per-element source records, the near
  // field of the FMM the node-sharing source stream (p2p.cu)
  rc = poro ? launch_poro_prep(ctx, t, perm_in, D, sp)
       : mode == DDM_DIRECT ? launch_prep_sources(ctx, t, perm_in, D, ncomp, sp)
                            : launch_prep_stream(ctx, t, perm_in, D, ncomp, sp,
                                                 early && (ctx->world > 1 || noexch) && t->shard_up);
  if (rc) return rc;
  stage_end(ctx, DDM_ST_PREP, sp);

  if (mode == DDM_DIRECT) {
    stage_begin(ctx, DDM_ST_P2P, s);
    rc = poro ? launch_poro_direct(ctx, t, lo, hi, PP, y_user, y_sorted, s)
              : launch_direct(ctx, t, lo, hi, ncomp, gc, y_user, y_sorted, s);
    stage_end(ctx, DDM_ST_P2P, s);
    return rc;
  }

  // fork: the near field (P2P, throughput bound) runs on the low-priority
  // stream concurrently with the latency-bound far-field chain on the
  // high-priority stream; both only read `src` / D and write disjoint buffers.
  if (!early) {
    DDM_CUDA(ctx, cudaEventRecord(ctx->ev_fork, s));
    DDM_CUDA(ctx, cudaStreamWaitEvent(sf, ctx->ev_fork, 0));
    DDM_CUDA(ctx, cudaStreamWaitEvent(sn, ctx->ev_fork, 0));
  }

  // DDM_TIMING_SKIP=near|far (scripts/timeline.py only; the result is then
  // wrong): launch one side of the fork alone, to time the other's span
  static const int skip = [] {
    const char* e = getenv("DDM_TIMING_SKIP");
    return !e ? 0 : !strcmp(e, "near") ? 1 : !strcmp(e, "far") ? 2 : 0;
  }();
  // near field: P2P work items of the owned leaves
  const bool leaf_p2p = !poro && use_leaf_p2p();
  // X lists: the elastic series FMM expands the coarser
  // non-touching U leaves of a large target leaf into its local series (P2L,
  // on the near stream ahead of the P2P; the L2P waits for it) and the P2P
  // reads U minus X; the M2L adds the P2L series to the leaves' locals
  const bool use_x = leaf_p2p && !bb && t->nx > 0;
  if (use_x) {
    stage_begin(ctx, DDM_ST_P2L, sn);
    if ((rc = launch_p2l(ctx, t, perm_in, D, ncomp, sn))) return rc;
    stage_end(ctx, DDM_ST_P2L, sn);
    DDM_CUDA(ctx, cudaEventRecord(ctx->ev_p2l, sn));
  }
  stage_begin(ctx, DDM_ST_P2P, sn);
  rc = skip == 1  ? DDM_OK
       : poro     ? launch_poro_p2p(ctx, t, t->item_lo_owned, t->item_hi_owned, PP, sn)
       : leaf_p2p ? launch_p2p_leaf(ctx, t, gc, sn, use_x)
                  : launch_p2p(ctx, t, t->item_lo_owned, t->item_hi_owned, gc, sn);
  if (rc) return rc;
  stage_end(ctx, DDM_ST_P2P, sn);
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_near, sn));

  if (skip == 2) {
  } else if (bb) {
    if ((rc = launch_bb_far(ctx, t, bb_n, perm_in ? t->d_sorted : D, ncomp, gc, sf))) return rc;
  } else {
  // upward pass: P2M on all leaves, M2M level by level; on several ranks
  // sharded: this rank's leaves and complete cells, the
  // multipole all-gather (overlapping the near field on the other stream),
  // then the straddling cells on every rank
  const bool sharded = (ctx->world > 1 || noexch) && t->shard_up;
  const int scope = sharded ? kUpOwn : kUpFull;
  if ((rc = early ? launch_upward(ctx, t, perm_in, D, ncomp, pf, sf, scope)
                  : launch_upward(ctx, t, nullptr, perm_in ? t->d_sorted : D, ncomp, pf, sf,
                                  scope)))
    return rc;
  if (sharded) {
    if ((rc = launch_mpole_pack(ctx, t, ctx->rank, sf))) return rc;
    stage_begin(ctx, DDM_ST_COMM, sf);
    if (!noexch && (rc = allgather_mpole(ctx, t, sf))) return rc;
    stage_end(ctx, DDM_ST_COMM, sf);
    if ((rc = launch_mpole_unpack(ctx, t, ctx->rank, ctx->world, sf))) return rc;
    if ((rc = launch_upward(ctx, t, nullptr, nullptr, ncomp, pf, sf, kUpStrad))) return rc;
  }
  // downward pass: M2L of every cell of level >= 2, L2L level by level (cells
  // whose subtree holds owned targets)
  if (use_x) DDM_CUDA(ctx, cudaStreamWaitEvent(sf, ctx->ev_p2l, 0));
  if ((rc = launch_downward(ctx, t, sf, use_x))) return rc;
  // L2P of the owned leaves (far field at the targets), still on the far stream
  stage_begin(ctx, DDM_ST_L2P, sf);
  if ((rc = launch_l2p(ctx, t, ncomp, gc, pf, sf))) return rc;
  stage_end(ctx, DDM_ST_L2P, sf);
  }
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_far, sf));

  // join
  DDM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_near, 0));
  DDM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_far, 0));
  stage_begin(ctx, DDM_ST_FINAL, s);
  rc = leaf_p2p ? launch_finalize_near(ctx, t, lo, hi, y_user, y_sorted, s)
                : launch_finalize(ctx, t, lo, hi, ncomp, gc, pf, y_user, y_sorted, s);
  stage_end(ctx, DDM_ST_FINAL, s);
  return rc;
}

// Fast history sum:
//   r = sum_{m=1}^{h} A^(m) D^(h-m) = sum_{j=1}^{h+1} K(j dt) E_j,  E_j = D^(h+1-j) - D^(h-j)
// (reading R10).  Far field (V pairs, all separated beyond R_c((h+1) dt)): the
// far form is affine in tau and sum_j E_j = 0, so it is ONE far pass of the
// tau-linear weights at tau = dt on S = sum_j j E_j = sum_{k<h} D^k.  Near
// field: one multi-lag launch (poro_hist_near_kernel).  D_hist [h][n][3] user
// order; writes the owned rows into y_user and/or y_sorted.
int fmm_history(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt, int h,
                const double* D_hist, double* y_user, double* y_sorted, cudaStream_t s) {
  int rc = fmm_workspace(ctx, t, s);
  if (rc) return rc;
  const PoroParams PP = poro_params(mat, dt);
  if (t->nlevels > 2) {
    const double ctmax = PP.c * ((h + 1) * dt);
    const double smin = std::ldexp(t->W, -(t->nlevels - 1));
    const double sep = smin - 2.0 * t->a_max;
    if (sep <= 0 || sep * sep / (4.0 * ctmax) <= 40.0)
      return set_error(ctx, DDM_ERR_ARG,
                       "tree too fine for the poroelastic far field at the history's longest lag: "
                       "build it with min_leaf_side >= sqrt(160 c (h+1) dt) + 2 max(a)");
  }
  const bool cached = poro_hist_cache_update(ctx, t, mat, dt, h, s, &rc);
  if (rc) return rc;
  const int64_t n = t->n;
  double *Hs = nullptr, *Cs = nullptr, *Ctot = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&Hs, (size_t)n * (h + 2) * 3 * sizeof(double), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&Cs, (size_t)n * (h + 1) * 3 * sizeof(double), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&Ctot, (size_t)n * 3 * sizeof(double), s));
  rc = launch_poro_hist_gather(ctx, t, h, D_hist, Hs, Cs, Ctot, s);
  // source geometry records (the D fields hold S, unused by the near kernel)
  if (!rc) rc = launch_poro_prep(ctx, t, nullptr, Ctot, s);
  if (rc) return rc;
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_fork, s));
  cudaStream_t sf = ctx->serial ? s : ctx->s_hi, sn = ctx->serial ? s : ctx->s_lo;
  DDM_CUDA(ctx, cudaStreamWaitEvent(sf, ctx->ev_fork, 0));
  DDM_CUDA(ctx, cudaStreamWaitEvent(sn, ctx->ev_fork, 0));
  stage_begin(ctx, DDM_ST_P2P, sn);
  rc = cached ? launch_poro_hist_cached(ctx, t, h, Hs, sn)
              : launch_poro_hist_near(ctx, t, PP, h, dt, Hs, Cs, sn);
  if (rc) return rc;
  stage_end(ctx, DDM_ST_P2P, sn);
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_near, sn));
  PoroFar pf = poro_far(PP);
  pf.lin = 1;   // tau-linear weights only, at tau = dt
  const double gc = mat->G / (4.0 * M_PI * (1.0 - mat->nu));
  if ((rc = launch_upward(ctx, t, nullptr, Ctot, 3, pf, sf))) return rc;
  if ((rc = launch_downward(ctx, t, sf))) return rc;
  stage_begin(ctx, DDM_ST_L2P, sf);
  if ((rc = launch_l2p(ctx, t, 3, gc, pf, sf))) return rc;
  stage_end(ctx, DDM_ST_L2P, sf);
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_far, sf));
  DDM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_near, 0));
  DDM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_far, 0));
  stage_begin(ctx, DDM_ST_FINAL, s);
  rc = launch_finalize(ctx, t, t->own_el_lo, t->own_el_hi, 3, gc, pf, y_user, y_sorted, s);
  stage_end(ctx, DDM_ST_FINAL, s);
  cudaFreeAsync(Hs, s);
  cudaFreeAsync(Cs, s);
  cudaFreeAsync(Ctot, s);
  return rc;
}

// Several ranks emulated on one device (tests): the elastic FMM
// matvec of the sharded path for trees[r] partitioned as rank r of `world`,
// every phase run rank by rank on stream s, with device copies standing in
// for the two NCCL all-gathers (multipoles, owned output rows).  Writes the
// full y in user order.
int fmm_matvec_sim(ddm_ctx_s* ctx, ddm_tree_s* const* trees, int world, const ddm_material* mat,
                   const double* D, double* y, cudaStream_t s) {
  int rc;
  if (world < 1) return set_error(ctx, DDM_ERR_ARG, "world < 1");
  if (mat->kind != 0) return set_error(ctx, DDM_ERR_ARG, "the emulation is elastic only");
  ddm_tree_s* t0 = trees[0];
  for (int r = 0; r < world; ++r) {
    ddm_tree_s* t = trees[r];
    if (t->n != t0->n || t->ncells != t0->ncells || t->p != t0->p || (int)t->xr_off.size() != world + 1 ||
        t->own_leaf_lo != t->rank_leaf_lo[r])
      return set_error(ctx, DDM_ERR_ARG, "trees[r] must be one geometry partitioned as rank r of world");
    if ((rc = fmm_workspace(ctx, t, s))) return rc;
  }
  const double gc = mat->G / (4.0 * M_PI * (1.0 - mat->nu));
  const PoroFar pf;
  const bool use_x = t0->nx > 0 && use_leaf_p2p();
  for (int r = 0; r < world; ++r) {   // phase A: near field, local upward pass, pack
    ddm_tree_s* t = trees[r];
    if ((rc = launch_prep_stream(ctx, t, t->perm, D, 2, s, world > 1))) return rc;
    if (use_x && (rc = launch_p2l(ctx, t, t->perm, D, 2, s))) return rc;
    if ((rc = launch_p2p_leaf(ctx, t, gc, s, use_x))) return rc;
    if ((rc = launch_upward(ctx, t, t->perm, D, 2, pf, s, world > 1 ? kUpOwn : kUpFull))) return rc;
    if (world > 1 && (rc = launch_mpole_pack(ctx, t, r, s))) return rc;
  }
  const size_t P2 = 2 * (size_t)t0->p;
  for (int r = 0; r < world && world > 1; ++r)   // the multipole all-gather
    for (int q = 0; q < world; ++q) {
      const int nc = trees[q]->xr_off[q + 1] - trees[q]->xr_off[q];
      if (nc > 0)
        DDM_CUDA(ctx, cudaMemcpyAsync(trees[r]->xrecv + (size_t)q * trees[r]->xr_max * P2,
                                      trees[q]->xsend, nc * P2 * sizeof(double2),
                                      cudaMemcpyDeviceToDevice, s));
    }
  double* ys = t0->y_sorted;
  for (int r = 0; r < world; ++r) {   // phase B: straddling cells, downward pass, assembly
    ddm_tree_s* t = trees[r];
    if (world > 1) {
      if ((rc = launch_mpole_unpack(ctx, t, r, world, s))) return rc;
      if ((rc = launch_upward(ctx, t, nullptr, nullptr, 2, pf, s, kUpStrad))) return rc;
    }
    if ((rc = launch_downward(ctx, t, s, use_x))) return rc;
    if ((rc = launch_l2p(ctx, t, 2, gc, pf, s))) return rc;
    // owned rows straight into the shared sorted vector (the row all-gather)
    if ((rc = launch_finalize_near(ctx, t, t->own_el_lo, t->own_el_hi, nullptr, ys, s))) return rc;
  }
  return launch_scatter_user(ctx, t0, ys, 2, y, s);
}

}  // namespace ddm
