// FMM matvec driver for the elastic constant-DD kernel and the
// host-side construction of the (scale-free) translation operators.
//
// PAPER.md §3.2: upward pass (P2M "P2L", M2M), downward pass (M2L
// over interaction lists, L2L), final L2P + P2P for self and neighbour cells.
// The paper's Chebyshev interpolation (bbFMM) is replaced by complex-variable
// (Kolosov–Muskhelishvili) expansions of the constant-element influence.
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

int ensure_workspace(ddm_ctx_s* ctx, ddm_tree_s* t) {
  int rc;
  if (!t->mpole) {
    if ((rc = dalloc(ctx, &t->mpole, (size_t)t->ncells * 2 * t->p))) return rc;
    if ((rc = dalloc(ctx, &t->local, (size_t)t->ncells * 2 * t->p))) return rc;
    if ((rc = dalloc(ctx, &t->src, (size_t)t->n * kSrcStride))) return rc;
    if ((rc = dalloc(ctx, &t->part, (size_t)t->nitems * kTgtGroup * 2))) return rc;  // <= 4 doubles/slot
    if ((rc = dalloc(ctx, &t->d_sorted, (size_t)t->n * 3))) return rc;
    if ((rc = dalloc(ctx, &t->y_sorted, (size_t)t->n * 3))) return rc;
  }
  return DDM_OK;
}

}  // namespace

// Translation operators (host, fp64), uploaded once per tree:
//   M2M_q[m][n] = 2^-n C(m-1, n-1) eps^(m-n)   (n <= m), eps = (z_q - z_P)/s_P
//   L2L_q[k][m] = C(m, k) 2^-k eps^(m-k)         (m >= k)
//   M2L: rot[o][k] = e^{-i k theta}, R[o][k] = (k-1)! rho^-k for the 49 offset
//        classes o = (dy+3)*7 + (dx+3), delta = -(dx + i dy) = rho e^{i theta}
// stored transposed ([n][m] resp. [m][k]) for coalesced lane = output access.
int fmm_init_operators(ddm_tree_s* t, cudaStream_t s) {
  ddm_ctx_s* ctx = t->ctx;
  const int p = t->p;
  typedef std::vector<double2> V;
  V m2m((size_t)4 * p * p), l2l((size_t)4 * p * p);
  auto cpow = [](double re, double im, int k) {
    double a = 1.0, b = 0.0;
    for (int i = 0; i < k; ++i) {
      const double na = a * re - b * im, nb = a * im + b * re;
      a = na;
      b = nb;
    }
    return make_double2(a, b);
  };
  for (int q = 0; q < 4; ++q) {
    const double ex_ = 0.5 * ((q & 1) - 0.5), ey_ = 0.5 * ((q >> 1) - 0.5);
    for (int m = 1; m <= p; ++m)
      for (int n = 1; n <= p; ++n) {
        double2 v = make_double2(0.0, 0.0);
        if (n <= m) {
          const double2 e = cpow(ex_, ey_, m - n);
          const double f = std::ldexp(1.0, -n) * binom(m - 1, n - 1);
          v = make_double2(f * e.x, f * e.y);
        }
        m2m[(size_t)q * p * p + (size_t)(n - 1) * p + (m - 1)] = v;
      }
    for (int k = 0; k < p; ++k)
      for (int m = 0; m < p; ++m) {
        double2 v = make_double2(0.0, 0.0);
        if (m >= k) {
          const double2 e = cpow(ex_, ey_, m - k);
          const double f = std::ldexp(1.0, -k) * binom(m, k);
          v = make_double2(f * e.x, f * e.y);
        }
        l2l[(size_t)q * p * p + (size_t)m * p + k] = v;
      }
  }
  std::vector<double> R((size_t)kNOffsets * (2 * p + 2), 0.0);
  V rot((size_t)kNOffsets * (p + 2), make_double2(0.0, 0.0));
  for (int o = 0; o < kNOffsets; ++o) {
    const int dx = o % 7 - 3, dy = o / 7 - 3;
    if (std::max(std::abs(dx), std::abs(dy)) < 2) continue;
    const double rho = std::sqrt((double)dx * dx + (double)dy * dy);
    const double er = -dx / rho, ei = dy / rho;   // e^{-i theta} = conj(delta)/rho
    double pr = 1.0, pi = 0.0;
    for (int k = 0; k < p + 2; ++k) {
      rot[(size_t)o * (p + 2) + k] = make_double2(pr, pi);
      const double nr = pr * er - pi * ei, ni = pr * ei + pi * er;
      pr = nr;
      pi = ni;
    }
    double fact = 1.0, rp = 1.0;
    for (int k = 1; k <= 2 * p + 1; ++k) {
      if (k >= 2) fact *= (k - 1);
      rp /= rho;
      R[(size_t)o * (2 * p + 2) + k] = fact * rp;
    }
  }
  std::vector<double> inv(2 * p + 2);
  double f = 1.0;
  for (int k = 0; k < 2 * p + 2; ++k) {
    if (k >= 1) f *= k;
    inv[k] = 1.0 / f;
  }
  int rc;
  if ((rc = dalloc(ctx, &t->op_m2m, m2m.size())) || (rc = dalloc(ctx, &t->op_l2l, l2l.size())) ||
      (rc = dalloc(ctx, &t->op_h, rot.size())) || (rc = dalloc(ctx, &t->invfact, inv.size())) ||
      (rc = dalloc(ctx, &t->op_R, R.size())))
    return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_R, R.data(), R.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_m2m, m2m.data(), m2m.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_l2l, l2l.data(), l2l.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->op_h, rot.data(), rot.size() * sizeof(double2),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->invfact, inv.data(), inv.size() * sizeof(double),
                                cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  return DDM_OK;
}

// Matvec y = A(elapsed) D.  D: [n][ncomp], user order
// (d_sorted = false) or sorted order, full length on every rank; ncomp = 2
// elastic, 3 poroelastic.  Writes the owned rows into y_user (user order)
// and/or y_sorted (sorted order).
int fmm_matvec(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double elapsed,
               const double* D, bool d_sorted, double* y_user, double* y_sorted, int mode,
               cudaStream_t s) {
  int rc = ensure_workspace(ctx, t);
  if (rc) return rc;
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

  stage_begin(ctx, DDM_ST_PREP, s);
  rc = poro ? launch_poro_prep(ctx, t, perm_in, D, s)
            : launch_prep_sources(ctx, t, perm_in, D, ncomp, s);
  if (rc) return rc;
  stage_end(ctx, DDM_ST_PREP, s);

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
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_fork, s));
  cudaStream_t sf = ctx->serial ? s : ctx->s_hi, sn = ctx->serial ? s : ctx->s_lo;
  DDM_CUDA(ctx, cudaStreamWaitEvent(sf, ctx->ev_fork, 0));
  DDM_CUDA(ctx, cudaStreamWaitEvent(sn, ctx->ev_fork, 0));

  // near field: P2P work items of the owned leaves
  stage_begin(ctx, DDM_ST_P2P, sn);
  rc = poro ? launch_poro_p2p(ctx, t, t->item_lo_owned, t->item_hi_owned, PP, sn)
            : launch_p2p(ctx, t, t->item_lo_owned, t->item_hi_owned, gc, sn);
  if (rc) return rc;
  stage_end(ctx, DDM_ST_P2P, sn);
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_near, sn));

  // upward pass (one persistent launch): P2M on all leaves + M2M finest ->
  // level 2, replicated on all ranks.  Stage "p2m" times the whole upward pass.
  stage_begin(ctx, DDM_ST_P2M, sf);
  if ((rc = launch_upward(ctx, t, perm_in, D, ncomp, pf, sf))) return rc;
  stage_end(ctx, DDM_ST_P2M, sf);

  // downward pass (one persistent launch): M2L + L2L of every cell of level
  // >= 2 whose subtree holds owned targets.  Stage "m2l" times the whole pass.
  stage_begin(ctx, DDM_ST_M2L, sf);
  if ((rc = launch_downward(ctx, t, sf))) return rc;
  stage_end(ctx, DDM_ST_M2L, sf);
  DDM_CUDA(ctx, cudaEventRecord(ctx->ev_far, sf));

  // join
  DDM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_near, 0));
  DDM_CUDA(ctx, cudaStreamWaitEvent(s, ctx->ev_far, 0));
  stage_begin(ctx, DDM_ST_FINAL, s);
  rc = launch_finalize(ctx, t, lo, hi, ncomp, gc, pf, y_user, y_sorted, s);
  stage_end(ctx, DDM_ST_FINAL, s);
  return rc;
}

}  // namespace ddm
