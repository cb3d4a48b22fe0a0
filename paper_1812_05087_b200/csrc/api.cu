// C-ABI entry points of libddm (include/ddm.h): context, tree, matvec,
// history, GMRES, loads, SIF, multi-GPU exchange.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <chrono>
#include <cstring>
#include <new>

#include "kcommon.cuh"

namespace ddm {

int set_error(ddm_ctx_s* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

int cuda_error_if(ddm_ctx_s* ctx, cudaError_t e, const char* what) {
  return e == cudaSuccess ? DDM_OK : cuda_error(ctx, e, what);
}

int cuda_error(ddm_ctx_s* ctx, cudaError_t e, const char* what) {
  cudaGetLastError();
  return set_error(ctx, e == cudaErrorMemoryAllocation ? DDM_ERR_OOM : DDM_ERR_CUDA,
                   std::string(what) + ": " + cudaGetErrorString(e));
}

void stage_begin(ddm_ctx_s* ctx, int st, cudaStream_t s) {
  if (ctx->profiling) cudaEventRecord(ctx->stage.ev[2 * st], s);
}
void stage_end(ddm_ctx_s* ctx, int st, cudaStream_t s) {
  if (ctx->profiling) cudaEventRecord(ctx->stage.ev[2 * st + 1], s);
}

namespace {

__global__ void unpack_allgather(const double* __restrict__ recv, const int64_t* __restrict__ lo,
                                 int world, int64_t maxrows, int ncomp, double* __restrict__ out) {
  const int r = blockIdx.y;
  const int64_t rows = lo[r + 1] - lo[r];
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < rows * ncomp;
       i += (int64_t)gridDim.x * blockDim.x)
    out[lo[r] * ncomp + i] = recv[r * maxrows * ncomp + i];
}

__global__ void scatter_user(int64_t n, int ncomp, const int* __restrict__ perm,
                             const double* __restrict__ ys, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm[i];
  for (int c = 0; c < ncomp; ++c) y[(int64_t)j * ncomp + c] = ys[i * ncomp + c];
}

__global__ void farfield_kernel(const double* __restrict__ beta, int64_t n, int ncomp, double pf,
                                double sH, double sh, int net, double bp, double* __restrict__ b) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double sb, cb;
  sincos(beta[i], &sb, &cb);
  const double sn_ff = sH * sb * sb + sh * cb * cb;
  b[i * ncomp + 0] = (sH - sh) * sb * cb;
  b[i * ncomp + 1] = net ? pf : pf - sn_ff;
  if (ncomp == 3) b[i * ncomp + 2] = bp;
}

__global__ void sif_kernel(const double* __restrict__ w, const double* __restrict__ ds,
                           const double* __restrict__ a, int n, double E, double nu,
                           double* __restrict__ KI, double* __restrict__ KII) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double f = 0.806 * E / (4.0 * (1.0 - nu * nu)) * sqrt(M_PI / (2.0 * a[i]));
  KI[i] = f * w[i];
  KII[i] = f * ds[i];
}

// DFMA throughput probe: 8 independent FMA chains per thread.
// Maximum-tangential-stress growth of one tip (ddm_tip_growth, reading R23)
__global__ void tip_growth_kernel(int ntips, const double* __restrict__ KI,
                                  const double* __restrict__ KII, const double* __restrict__ x,
                                  const double* __restrict__ y, const double* __restrict__ a,
                                  const double* __restrict__ beta, const int* __restrict__ end,
                                  double kic, int* __restrict__ grow, double* __restrict__ nx,
                                  double* __restrict__ ny, double* __restrict__ na,
                                  double* __restrict__ nb, int* __restrict__ ne) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ntips) return;
  const double k1 = KI[i], k2 = KII[i];
  const double th = k2 == 0.0 ? 0.0 : 2.0 * atan((k1 - sqrt(k1 * k1 + 8.0 * k2 * k2)) / (4.0 * k2));
  const double ch = cos(0.5 * th);
  const double keq = ch * (k1 * ch * ch - 1.5 * k2 * sin(th));
  const int g = (k1 > 0.0 && keq >= kic) ? 1 : 0;
  grow[i] = g;
  if (!g) return;
  const double b = beta[i], ai = a[i];
  const double sgn = end[i] ? 1.0 : -1.0;
  const double ex = x[i] + sgn * ai * cos(b), ey = y[i] + sgn * ai * sin(b);   // tip point
  double phi = (end[i] ? b : b + M_PI) + th;                                   // growth direction
  phi = fmod(phi, 2.0 * M_PI);
  if (phi < 0.0) phi += 2.0 * M_PI;
  nx[i] = ex + ai * cos(phi);
  ny[i] = ey + ai * sin(phi);
  na[i] = ai;
  // beta in [0, pi); the outward end is + e^{i beta} when phi < pi
  const bool up = phi < M_PI;
  nb[i] = up ? phi : phi - M_PI;
  ne[i] = up ? 1 : 0;
}

__global__ void dfma_probe_kernel(int iters, double a, double b, double* out) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0.0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  if (s == 1.2345e-300) out[0] = s;   // keep the chains alive
}

int check_material(ddm_ctx_s* ctx, const ddm_material* m) {
  if (!m) return set_error(ctx, DDM_ERR_ARG, "material is NULL");
  if (m->kind != 0 && m->kind != 1) return set_error(ctx, DDM_ERR_ARG, "material kind not 0/1");
  if (!(m->G > 0) || !(m->nu > -1.0 && m->nu < 0.5))
    return set_error(ctx, DDM_ERR_ARG, "material needs G > 0 and -1 < nu < 0.5");
  if (m->kind == 1 && !(m->nu_u > m->nu && m->nu_u < 0.5 && m->alpha > 0 && m->alpha <= 1 &&
                        m->kappa > 0))
    return set_error(ctx, DDM_ERR_ARG, "poroelastic material needs nu < nu_u < 0.5, 0 < alpha <= 1, kappa > 0");
  return DDM_OK;
}

}  // namespace

// all-gather of the owned sorted rows y_sorted[lo..hi) into the full vector
// (persistent buffers from the partition: no allocation per call)
int allgather_sorted(ddm_ctx_s* ctx, ddm_tree_s* t, double* buf, int ncomp, cudaStream_t s) {
  if (!ctx->exchange) return DDM_OK;
#ifdef DDM_WITH_NCCL
  if (!t->ag_send) return set_error(ctx, DDM_ERR_ARG, "tree not partitioned for the exchange");
  const int64_t maxrows = t->ag_max;
  const size_t cnt = (size_t)maxrows * ncomp;
  const int64_t lo = t->own_el_lo, hi = t->own_el_hi;
  if (hi > lo)
    DDM_CUDA(ctx, cudaMemcpyAsync(t->ag_send, buf + lo * ncomp, (hi - lo) * ncomp * sizeof(double),
                                  cudaMemcpyDeviceToDevice, s));
  ncclResult_t nr = ncclAllGather(t->ag_send, t->ag_recv, cnt, ncclDouble, ctx->comm, s);
  if (nr != ncclSuccess)
    return set_error(ctx, DDM_ERR_NCCL, std::string("ncclAllGather: ") + ncclGetErrorString(nr));
  dim3 grid(std::max(1u, nblk(maxrows * ncomp, 256)), ctx->world);
  unpack_allgather<<<grid, 256, 0, s>>>(t->ag_recv, t->ag_lo, ctx->world, maxrows, ncomp, buf);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
#else
  (void)t; (void)buf; (void)ncomp; (void)s;
  return set_error(ctx, DDM_ERR_NCCL, "libddm built without NCCL");
#endif
}

// all-gather of the packed multipoles of every rank's complete cells (the
// sharded upward pass), padded to xr_max cells per rank
int allgather_mpole(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s) {
#ifdef DDM_WITH_NCCL
  const size_t cnt = (size_t)t->xr_max * 2 * t->p * 2;   // doubles
  if (cnt == 0) return DDM_OK;
  ncclResult_t nr = ncclAllGather(t->xsend, t->xrecv, cnt, ncclDouble, ctx->comm, s);
  if (nr != ncclSuccess)
    return set_error(ctx, DDM_ERR_NCCL, std::string("ncclAllGather (multipoles): ") +
                                            ncclGetErrorString(nr));
  return DDM_OK;
#else
  (void)t; (void)s;
  return set_error(ctx, DDM_ERR_NCCL, "libddm built without NCCL");
#endif
}

int launch_scatter_user(ddm_ctx_s* ctx, ddm_tree_s* t, const double* ys, int ncomp, double* y,
                        cudaStream_t s) {
  scatter_user<<<nblk(t->n, 256), 256, 0, s>>>(t->n, ncomp, t->perm, ys, y);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int allreduce_sum(ddm_ctx_s* ctx, double* buf, int64_t count, cudaStream_t s) {
  if (!ctx->exchange) return DDM_OK;
#ifdef DDM_WITH_NCCL
  ncclResult_t nr = ncclAllReduce(buf, buf, (size_t)count, ncclDouble, ncclSum, ctx->comm, s);
  if (nr != ncclSuccess)
    return set_error(ctx, DDM_ERR_NCCL, std::string("ncclAllReduce: ") + ncclGetErrorString(nr));
  return DDM_OK;
#else
  (void)buf; (void)count; (void)s;
  return set_error(ctx, DDM_ERR_NCCL, "libddm built without NCCL");
#endif
}

// Everything derived from the owned range (captured matvec graphs, the
// near-field and history caches of the owned items, the owned preconditioner
// chunks) is dropped when the partition changes; it is rebuilt on demand.
static void drop_owned_state(ddm_tree_s* t) {
  drop_graphs(t);
  {
    void* sh[] = {t->xr_cells, t->xr_off_dev, t->up_own, t->up_strad, t->xsend, t->xrecv,
                  t->ag_send, t->ag_recv, t->ag_lo, t->halo_rng, t->halo_pre, t->dn_own};
    t->dn_own = nullptr;
    if (t->l2p_runs) cudaFree(t->l2p_runs);
    if (t->l2p_order) cudaFree(t->l2p_order);
    if (t->p2p_leaf_order) cudaFree(t->p2p_leaf_order);
    t->p2p_leaf_order = nullptr;
    t->p2m_own_lo = t->p2m_own_hi = -1;
    t->l2p_runs = nullptr;
    t->l2p_order = nullptr;
    t->l2p_nruns = 0;
    t->l2p_lo = t->l2p_hi = -1;
    t->halo_rng = nullptr;
    t->halo_pre = nullptr;
    t->nhalo = 0;
    t->halo_slots = 0;
    for (void* p : sh)
      if (p) cudaFree(p);
    t->xr_cells = nullptr;
    t->xr_off_dev = nullptr;
    t->up_own = t->up_strad = nullptr;
    t->xsend = t->xrecv = nullptr;
    t->ag_send = t->ag_recv = nullptr;
    t->ag_lo = nullptr;
    t->xr_max = 0;
    t->ag_max = 0;
    t->shard_up = false;
  }
  for (double* p : t->hc_alloc) cudaFree(p);
  t->hc_alloc.clear();
  t->hc_lag.clear();
  t->hc_nlags = 0;
  t->hc_valid = t->hc_seen_set = t->hc_capped = false;
  void* ptrs[] = {t->nc, t->nc_off, t->pc_chunks, t->pc_off, t->pcl};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  t->nc = nullptr;
  t->nc_off = nullptr;
  t->nc_n = 0;
  t->nc_valid = t->nc_seen_set = false;
  t->pc_chunks = nullptr;
  t->pc_off = nullptr;
  t->pcl = nullptr;
  t->pc_nchunks = t->pc_off_ncomp = 0;
  std::memset(t->pcl_key, 0, sizeof(t->pcl_key));
}

void shard_owner(const int* c_start, const int* c_count, int ncells, const int64_t* lo, int world,
                 int* owner) {
  for (int c = 0; c < ncells; ++c) {
    const int64_t a = c_start[c], b = a + c_count[c];
    // the rank whose range contains the cell's first element
    const int r = (int)(std::upper_bound(lo, lo + world + 1, a) - lo) - 1;
    owner[c] = (r >= 0 && r < world && a >= lo[r] && b <= lo[r + 1]) ? r : -1;
  }
}

// Sharded upward pass metadata and the persistent exchange
// buffers: per rank the cells whose element range lies inside its range
// (complete cells), this rank's complete non-leaf cells and the straddling
// non-leaf cells as per-level M2M lists (deepest level first).
static int shard_metadata(ddm_tree_s* t, int rank, int world, const std::vector<int>& h_start,
                          cudaStream_t s) {
  ddm_ctx_s* ctx = t->ctx;
  const int nc = t->ncells;
  std::vector<int> h_count(nc);
  DDM_CUDA(ctx, cudaMemcpyAsync(h_count.data(), t->c_count, nc * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  const std::vector<int64_t>& lo = t->rank_el_lo;
  std::vector<int> owner(nc, -1);
  shard_owner(h_start.data(), h_count.data(), nc, lo.data(), world, owner.data());
  std::vector<std::vector<int>> per(world);
  for (int c = 0; c < nc; ++c)
    if (owner[c] >= 0) per[owner[c]].push_back(c);
  std::vector<int> cells;
  t->xr_off.assign(world + 1, 0);
  t->xr_max = 0;
  for (int r = 0; r < world; ++r) {
    t->xr_off[r] = (int)cells.size();
    cells.insert(cells.end(), per[r].begin(), per[r].end());
    t->xr_max = std::max(t->xr_max, (int)per[r].size());
  }
  t->xr_off[world] = (int)cells.size();
  std::vector<int> own, strad;
  t->up_own_off.assign(2 * (t->nlevels + 1), 0);
  t->up_strad_off.assign(2 * (t->nlevels + 1), 0);
  for (int lev = t->nlevels - 1; lev >= 2; --lev) {
    t->up_own_off[2 * lev] = (int)own.size();
    t->up_strad_off[2 * lev] = (int)strad.size();
    for (int k = t->up_level_off[2 * lev]; k < t->up_level_off[2 * lev + 1]; ++k) {
      const int c = t->h_up[k];
      if (owner[c] == rank) own.push_back(c);
      else if (owner[c] < 0) strad.push_back(c);
    }
    t->up_own_off[2 * lev + 1] = (int)own.size();
    t->up_strad_off[2 * lev + 1] = (int)strad.size();
  }
  t->shard_up = world > 1;
  int rc0;
  // downward-pass cell list of this rank (cells whose range meets the owned range)
  std::vector<int> dn;
  t->dn_own_off.assign(t->nlevels + 1, 0);
  for (int lev = 0; lev < t->nlevels; ++lev) {
    t->dn_own_off[lev] = (int)dn.size();
    if (lev < 2) continue;
    for (int c = t->level_off[lev]; c < t->level_off[lev + 1]; ++c)
      if ((int64_t)h_start[c] < t->own_el_hi && (int64_t)h_start[c] + h_count[c] > t->own_el_lo)
        dn.push_back(c);
  }
  t->dn_own_off[t->nlevels] = (int)dn.size();
  if (world > 1) {
    if ((rc0 = dalloc(ctx, &t->dn_own, dn.size()))) return rc0;
    if (!dn.empty())
      DDM_CUDA(ctx, cudaMemcpyAsync(t->dn_own, dn.data(), dn.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, s));
  }
  // near-field halo: the slots of the owned leaves' U ranges, plus the slot
  // before them (its record carries the node of a linked first record)
  t->halo_lo = 0;
  t->halo_hi = t->n;
  if (world > 1) {
    const int l0 = t->own_leaf_lo, l1 = t->own_leaf_hi;
    if (l1 > l0) {
      std::vector<int> uoff(l1 - l0 + 1);
      DDM_CUDA(ctx, cudaMemcpyAsync(uoff.data(), t->u_off + l0, uoff.size() * sizeof(int),
                                    cudaMemcpyDeviceToHost, s));
      DDM_CUDA(ctx, cudaStreamSynchronize(s));
      const int r0 = uoff.front(), r1 = uoff.back();
      std::vector<int> ulo(std::max(r1 - r0, 1)), uhi(std::max(r1 - r0, 1));
      if (r1 > r0) {
        DDM_CUDA(ctx, cudaMemcpyAsync(ulo.data(), t->u_lo + r0, (r1 - r0) * sizeof(int),
                                      cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaMemcpyAsync(uhi.data(), t->u_hi + r0, (r1 - r0) * sizeof(int),
                                      cudaMemcpyDeviceToHost, s));
        DDM_CUDA(ctx, cudaStreamSynchronize(s));
        int64_t a = t->n, b = 0;
        std::vector<std::pair<int, int>> iv(r1 - r0);
        for (int k = 0; k < r1 - r0; ++k) {
          a = std::min<int64_t>(a, ulo[k]);
          b = std::max<int64_t>(b, uhi[k]);
          iv[k] = {std::max(0, ulo[k] - 1), uhi[k]};
        }
        t->halo_lo = std::max<int64_t>(0, a - 1);
        t->halo_hi = b;
        std::sort(iv.begin(), iv.end());
        std::vector<int2> mr;
        for (const auto& v : iv) {
          if (!mr.empty() && v.first <= mr.back().y) mr.back().y = std::max(mr.back().y, v.second);
          else mr.push_back(make_int2(v.first, v.second));
        }
        std::vector<int64_t> pre(mr.size() + 1, 0);
        for (size_t k = 0; k < mr.size(); ++k) pre[k + 1] = pre[k] + (mr[k].y - mr[k].x);
        t->nhalo = (int)mr.size();
        t->halo_slots = pre.back();
        if ((rc0 = dalloc(ctx, &t->halo_rng, mr.size())) || (rc0 = dalloc(ctx, &t->halo_pre, pre.size())))
          return rc0;
        DDM_CUDA(ctx, cudaMemcpyAsync(t->halo_rng, mr.data(), mr.size() * sizeof(int2),
                                      cudaMemcpyHostToDevice, s));
        DDM_CUDA(ctx, cudaMemcpyAsync(t->halo_pre, pre.data(), pre.size() * sizeof(int64_t),
                                      cudaMemcpyHostToDevice, s));
      }
    } else {
      t->halo_lo = t->halo_hi = 0;
    }
  }
  int rc;
  const size_t P2 = 2 * (size_t)t->p;
  if ((rc = dalloc(ctx, &t->xr_cells, cells.size())) || (rc = dalloc(ctx, &t->xr_off_dev, world + 1)) ||
      (rc = dalloc(ctx, &t->up_own, own.size())) || (rc = dalloc(ctx, &t->up_strad, strad.size())))
    return rc;
  if (world > 1 && ((rc = dalloc(ctx, &t->xsend, (size_t)std::max(t->xr_max, 1) * P2)) ||
                    (rc = dalloc(ctx, &t->xrecv, (size_t)std::max(t->xr_max, 1) * P2 * world))))
    return rc;
  if (!cells.empty())
    DDM_CUDA(ctx, cudaMemcpyAsync(t->xr_cells, cells.data(), cells.size() * sizeof(int),
                                  cudaMemcpyHostToDevice, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(t->xr_off_dev, t->xr_off.data(), (world + 1) * sizeof(int),
                                cudaMemcpyHostToDevice, s));
  if (!own.empty())
    DDM_CUDA(ctx, cudaMemcpyAsync(t->up_own, own.data(), own.size() * sizeof(int),
                                  cudaMemcpyHostToDevice, s));
  if (!strad.empty())
    DDM_CUDA(ctx, cudaMemcpyAsync(t->up_strad, strad.data(), strad.size() * sizeof(int),
                                  cudaMemcpyHostToDevice, s));
  // all-gather buffers of the owned output rows (<= 3 components)
  t->ag_max = 0;
  for (int r = 0; r < world; ++r) t->ag_max = std::max(t->ag_max, lo[r + 1] - lo[r]);
  if (world > 1 || ctx->exchange) {
  if ((rc = dalloc(ctx, &t->ag_send, (size_t)std::max<int64_t>(t->ag_max, 1) * 3)) ||
      (rc = dalloc(ctx, &t->ag_recv, (size_t)std::max<int64_t>(t->ag_max, 1) * 3 * world)) ||
      (rc = dalloc(ctx, &t->ag_lo, world + 1)))
    return rc;
  DDM_CUDA(ctx, cudaMemcpyAsync(t->ag_lo, lo.data(), (world + 1) * sizeof(int64_t),
                                cudaMemcpyHostToDevice, s));
  }
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  return DDM_OK;
}

int partition_tree(ddm_tree_s* t, int rank, int world, cudaStream_t s) {
  ddm_ctx_s* ctx = t->ctx;
  int rc0;
  if (world < 1 || rank < 0 || rank >= world)
    return set_error(ctx, DDM_ERR_ARG, "bad rank/world");
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  drop_owned_state(t);
  std::vector<int> split(world + 1);
  split_costs(t->leaf_cost_prefix.data(), t->leaf_cost_prefix[t->nleaves], t->nleaves, world,
              split.data());
  t->rank_leaf_lo = split;
  // element and item boundaries of each rank's leaf range
  std::vector<int> h_leaves(t->nleaves), h_start(t->ncells), h_ioff(t->nleaves + 1);
  DDM_CUDA(ctx, cudaMemcpyAsync(h_leaves.data(), t->leaves, t->nleaves * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(h_start.data(), t->c_start, t->ncells * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(h_ioff.data(), t->item_off, (t->nleaves + 1) * sizeof(int),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  t->rank_el_lo.assign(world + 1, 0);
  for (int r = 0; r < world; ++r)
    t->rank_el_lo[r] = split[r] < t->nleaves ? h_start[h_leaves[split[r]]] : t->n;
  t->rank_el_lo[world] = t->n;
  t->own_leaf_lo = split[rank];
  t->own_leaf_hi = split[rank + 1];
  t->own_el_lo = t->rank_el_lo[rank];
  t->own_el_hi = t->rank_el_lo[rank + 1];
  t->item_lo_owned = h_ioff[split[rank]];
  t->item_hi_owned = h_ioff[split[rank + 1]];
  if ((rc0 = shard_metadata(t, rank, world, h_start, s))) return rc0;
  // execution order of the owned P2P items: Morton order (consecutive warps
  // share source records in L2; measured: a longest-first order doubled the
  // DRAM traffic of p2p_kernel for no time gain -- items are capped at
  // kSrcChunk sources, so there is no long tail to schedule first)
  const int nown = t->item_hi_owned - t->item_lo_owned;
  if (t->p2p_order) cudaFree(t->p2p_order);
  t->p2p_order = nullptr;
  if (nown > 0) {
    std::vector<int> order(nown);
    for (int i = 0; i < nown; ++i) order[i] = t->item_lo_owned + i;
    int rc = dalloc(ctx, &t->p2p_order, nown);
    if (rc) return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->p2p_order, order.data(), nown * sizeof(int),
                                  cudaMemcpyHostToDevice, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
  }
  return DDM_OK;
}

}  // namespace ddm

using namespace ddm;

extern "C" {

const char* ddm_version(void) { return "ddm-b200 0.1 sm_100a fp64"; }

const char* ddm_last_error(ddm_ctx_t ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int ddm_nccl_unique_id(void* uid_out) {
#ifdef DDM_WITH_NCCL
  if (!uid_out) return DDM_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return DDM_ERR_NCCL;
  std::memcpy(uid_out, &id, sizeof(id));
  return DDM_OK;
#else
  (void)uid_out;
  return DDM_ERR_NCCL;
#endif
}

int ddm_ctx_create(int device, const void* nccl_uid, int rank, int world, ddm_ctx_t* out) {
  if (!out) return DDM_ERR_ARG;
  *out = nullptr;
  if (world < 1 || rank < 0 || rank >= world) return DDM_ERR_ARG;
  ddm_ctx_s* ctx = new (std::nothrow) ddm_ctx_s();
  if (!ctx) return DDM_ERR_OOM;
  ctx->device = device;
  ctx->rank = rank;
  ctx->world = world;
  cudaError_t e = cudaSetDevice(device);
  if (e != cudaSuccess) {
    int rc = cuda_error(ctx, e, "cudaSetDevice");
    *out = ctx;
    return rc;
  }
  {
    // stream-ordered workspaces (cudaMallocAsync in history / GMRES calls)
    // stay mapped in the device's default pool between calls instead of
    // being unmapped at every synchronisation and remapped by the next call
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
      uint64_t keep = UINT64_MAX;
      cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
    }
  }
  e = cudaMalloc((void**)&ctx->d_scalar, 64 * sizeof(double));
  if (e != cudaSuccess) {
    int rc = cuda_error(ctx, e, "cudaMalloc(scratch)");
    *out = ctx;
    return rc;
  }
  {
    int rc = poro_init_tables(ctx);
    if (rc) {
      *out = ctx;
      return rc;
    }
  }
  {
    const char* ser = getenv("DDM_SERIAL");
    ctx->serial = ctx->serial_env = ser && ser[0] == '1';
    int lo_prio = 0, hi_prio = 0;
    cudaDeviceGetStreamPriorityRange(&lo_prio, &hi_prio);
    if (const char* sw = getenv("DDM_PRIO_SWAP"))   // experiment: near field high priority
      if (sw[0] == '1') std::swap(lo_prio, hi_prio);
    if ((e = cudaStreamCreateWithPriority(&ctx->s_hi, cudaStreamNonBlocking, hi_prio)) != cudaSuccess ||
        (e = cudaStreamCreateWithPriority(&ctx->s_lo, cudaStreamNonBlocking, lo_prio)) != cudaSuccess ||
        (e = cudaStreamCreateWithFlags(&ctx->s_cap, cudaStreamNonBlocking)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_fork, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_far, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_near, cudaEventDisableTiming)) != cudaSuccess ||
        (e = cudaEventCreateWithFlags(&ctx->ev_p2l, cudaEventDisableTiming)) != cudaSuccess) {
      int rc = cuda_error(ctx, e, "stream/event creation");
      *out = ctx;
      return rc;
    }
  }
  const bool force_nccl = [] {
    const char* e = getenv("DDM_FORCE_NCCL");
    return e && e[0] == '1';
  }();
  if (world > 1 || force_nccl) {
#ifdef DDM_WITH_NCCL
    ncclUniqueId id;
    if (world == 1) {   // one-rank communicator (exchange path test)
      if (ncclGetUniqueId(&id) != ncclSuccess) {
        *out = ctx;
        return set_error(ctx, DDM_ERR_NCCL, "ncclGetUniqueId");
      }
    } else {
      if (!nccl_uid) {
        *out = ctx;
        return set_error(ctx, DDM_ERR_ARG, "world > 1 needs an ncclUniqueId");
      }
      std::memcpy(&id, nccl_uid, sizeof(id));
    }
    ctx->exchange = true;
    ncclResult_t nr = ncclCommInitRank(&ctx->comm, world, id, rank);
    if (nr != ncclSuccess) {
      *out = ctx;
      return set_error(ctx, DDM_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(nr));
    }
#else
    *out = ctx;
    return set_error(ctx, DDM_ERR_NCCL, "libddm built without NCCL");
#endif
  }
  *out = ctx;
  return DDM_OK;
}

void ddm_ctx_destroy(ddm_ctx_t ctx) {
  if (!ctx) return;
#ifdef DDM_WITH_NCCL
  if (ctx->comm) ncclCommDestroy(ctx->comm);
#endif
  if (ctx->stage.created)
    for (auto& ev : ctx->stage.ev) cudaEventDestroy(ev);
  for (cudaEvent_t ev : {ctx->ev_fork, ctx->ev_far, ctx->ev_near, ctx->ev_p2l})
    if (ev) cudaEventDestroy(ev);
  for (cudaStream_t st : {ctx->s_hi, ctx->s_lo, ctx->s_cap})
    if (st) cudaStreamDestroy(st);
  if (ctx->d_scalar) cudaFree(ctx->d_scalar);
  if (ctx->h_pinned) cudaFreeHost(ctx->h_pinned);
  delete ctx;
}

int ddm_set_profiling(ddm_ctx_t ctx, int enable) {
  if (!ctx) return DDM_ERR_ARG;
  if (enable && !ctx->stage.created) {
    for (auto& ev : ctx->stage.ev) DDM_CUDA(ctx, cudaEventCreate(&ev));
    ctx->stage.created = true;
  }
  ctx->profiling = enable != 0;
  // mode 2: serial schedule, so every stage's events bracket that stage alone
  ctx->serial = enable == 2 ? true : ctx->serial_env;
  return DDM_OK;
}

int ddm_stage_times(ddm_ctx_t ctx, double* ms) {
  if (!ctx || !ms) return DDM_ERR_ARG;
  if (!ctx->profiling) return set_error(ctx, DDM_ERR_ARG, "profiling not enabled");
  // DDM_STAGE_ENDS=1 (scripts/timeline.py): each stage's END relative to the
  // start of prep instead of its duration -- the concurrent schedule's timeline
  static const bool ends = [] {
    const char* e = getenv("DDM_STAGE_ENDS");
    return e && e[0] == '1';
  }();
  for (int st = 0; st < DDM_NSTAGES; ++st) {
    float v = 0.f;
    if (cudaEventElapsedTime(&v, ctx->stage.ev[ends ? 2 * DDM_ST_PREP : 2 * st],
                             ctx->stage.ev[2 * st + 1]) != cudaSuccess) {
      cudaGetLastError();
      v = 0.f;
    }
    ms[st] = v;
  }
  return DDM_OK;
}

int ddm_build_tree(ddm_ctx_t ctx, const double* xc, const double* yc, const double* half_len,
                   const double* beta, int64_t n, int leaf_size, int order_p, double min_leaf_side,
                   void* stream, ddm_tree_t* out) {
  if (!ctx || !out) return DDM_ERR_ARG;
  *out = nullptr;
  if (!xc || !yc || !half_len || !beta) return set_error(ctx, DDM_ERR_ARG, "NULL geometry array");
  cudaStream_t s = (cudaStream_t)stream;
  ddm_tree_s* t = new (std::nothrow) ddm_tree_s();
  if (!t) return set_error(ctx, DDM_ERR_OOM, "host allocation");
  const auto t0 = std::chrono::steady_clock::now();
  int rc = build_tree(ctx, xc, yc, half_len, beta, n, leaf_size, order_p, min_leaf_side, s, t);
  if (!rc) rc = fmm_init_operators(t, s);
  if (!rc) rc = partition_tree(t, ctx->rank, ctx->world, s);
  t->build_ms[DDM_TB_TOTAL] =
      std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
  if (rc) {
    cudaStreamSynchronize(s);
    cudaGetLastError();
    free_tree(t);
    delete t;
    return rc;
  }
  *out = t;
  return DDM_OK;
}

void ddm_tree_free(ddm_tree_t t) {
  if (!t) return;
  cudaDeviceSynchronize();
  free_tree(t);
  delete t;
}

int ddm_tree_partition(ddm_tree_t t, int rank, int world) {
  if (!t) return DDM_ERR_ARG;
  return partition_tree(t, rank, world, 0);
}

int ddm_tree_counts(ddm_tree_t t, int64_t* c) {
  if (!t || !c) return DDM_ERR_ARG;
  for (int i = 0; i < DDM_TREE_NCOUNTS; ++i) c[i] = 0;
  c[DDM_TC_N] = t->n;
  c[DDM_TC_CELLS] = t->ncells;
  c[DDM_TC_LEAVES] = t->nleaves;
  c[DDM_TC_LEVELS] = t->nlevels;
  c[DDM_TC_V] = t->nv;
  c[DDM_TC_URANGES] = t->nu;
  c[DDM_TC_NEAR_PAIRS] = t->near_pairs;
  c[DDM_TC_P2P_ITEMS] = t->nitems;
  c[DDM_TC_OWNED_LO] = t->own_el_lo;
  c[DDM_TC_OWNED_HI] = t->own_el_hi;
  c[DDM_TC_P] = t->p;
  c[DDM_TC_W] = t->nw;
  c[DDM_TC_W_MIN] = t->w_min;
  c[DDM_TC_X] = t->nx;
  c[DDM_TC_X_MIN] = t->xl_min;
  c[DDM_TC_UXRANGES] = t->nux;
  c[DDM_TC_NEAR_PAIRS_P2P] = t->nx > 0 ? t->near_pairs_x : t->near_pairs;
  return DDM_OK;
}

int ddm_tree_build_times(ddm_tree_t t, double* ms) {
  if (!t || !ms) return DDM_ERR_ARG;
  for (int i = 0; i < DDM_TB_N; ++i) ms[i] = t->build_ms[i];
  return DDM_OK;
}

int ddm_tree_export(ddm_tree_t t, int what, void* dst, int64_t cap) {
  if (!t || !dst) return DDM_ERR_ARG;
  ddm_ctx_s* ctx = t->ctx;
  const void* src = nullptr;
  size_t bytes = 0;
  double root[3] = {t->x_min, t->y_min, t->W};
  const size_t nc = (size_t)t->ncells;
  switch (what) {
    case DDM_EX_KEYS: src = t->keys_user; bytes = t->n * 8; break;
    case DDM_EX_PERM: src = t->perm; bytes = t->n * 4; break;
    case DDM_EX_ROOT:
      if (cap < 24) return set_error(ctx, DDM_ERR_ARG, "capacity too small");
      std::memcpy(dst, root, 24);
      return DDM_OK;
    case DDM_EX_LEVEL: src = t->c_level; bytes = nc * 4; break;
    case DDM_EX_IX: src = t->c_ix; bytes = nc * 4; break;
    case DDM_EX_IY: src = t->c_iy; bytes = nc * 4; break;
    case DDM_EX_START: src = t->c_start; bytes = nc * 4; break;
    case DDM_EX_COUNT: src = t->c_count; bytes = nc * 4; break;
    case DDM_EX_PARENT: src = t->c_parent; bytes = nc * 4; break;
    case DDM_EX_FIRST_CHILD: src = t->c_first_child; bytes = nc * 4; break;
    case DDM_EX_NCHILD: src = t->c_nchild; bytes = nc * 4; break;
    case DDM_EX_LEAF: src = t->c_leaf; bytes = nc * 4; break;
    case DDM_EX_V_OFF: src = t->v_off; bytes = (nc + 1) * 4; break;
    case DDM_EX_V_IDX: src = t->v_idx; bytes = t->nv * 4; break;
    case DDM_EX_LEAVES: src = t->leaves; bytes = (size_t)t->nleaves * 4; break;
    case DDM_EX_U_OFF: src = t->u_off; bytes = ((size_t)t->nleaves + 1) * 4; break;
    case DDM_EX_U_LO: src = t->u_lo; bytes = t->nu * 4; break;
    case DDM_EX_U_HI: src = t->u_hi; bytes = t->nu * 4; break;
    case DDM_EX_W_OFF: src = t->w_off; bytes = ((size_t)t->nleaves + 1) * 4; break;
    case DDM_EX_W_IDX: src = t->w_idx; bytes = t->nw * 4; break;
    case DDM_EX_X_OFF: src = t->x_off; bytes = ((size_t)t->nleaves + 1) * 4; break;
    case DDM_EX_X_IDX: src = t->x_idx; bytes = t->nx * 4; break;
    case DDM_EX_UX_OFF: src = t->ux_off; bytes = ((size_t)t->nleaves + 1) * 4; break;
    case DDM_EX_UX_LO: src = t->ux_lo; bytes = t->nux * 4; break;
    case DDM_EX_UX_HI: src = t->ux_hi; bytes = t->nux * 4; break;
    default: return set_error(ctx, DDM_ERR_ARG, "unknown export id");
  }
  if ((int64_t)bytes > cap) return set_error(ctx, DDM_ERR_ARG, "capacity too small");
  if (bytes) DDM_CUDA(ctx, cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost));
  return DDM_OK;
}

int ddm_shard_owner(const int* c_start, const int* c_count, int ncells, const int64_t* rank_el_lo,
                    int world, int* owner) {
  if (!c_start || !c_count || !rank_el_lo || !owner || ncells < 0 || world < 1) return DDM_ERR_ARG;
  shard_owner(c_start, c_count, ncells, rank_el_lo, world, owner);
  return DDM_OK;
}

int ddm_matvec_sim(ddm_ctx_t ctx, const ddm_tree_t* trees, int world, const ddm_material* mat,
                   const double* D, double* y, void* stream) {
  if (!ctx || !trees || !D || !y || world < 1)
    return ctx ? set_error(ctx, DDM_ERR_ARG, "NULL argument") : DDM_ERR_ARG;
  int rc = check_material(ctx, mat);
  if (rc) return rc;
  for (int r = 0; r < world; ++r)
    if (!trees[r]) return set_error(ctx, DDM_ERR_ARG, "NULL tree");
  return fmm_matvec_sim(ctx, trees, world, mat, D, y, (cudaStream_t)stream);
}

int ddm_matvec(ddm_ctx_t ctx, ddm_tree_t t, const ddm_material* mat, double elapsed,
               const double* D, double* y, int mode, void* stream) {
  if (!ctx || !t || !D || !y) return ctx ? set_error(ctx, DDM_ERR_ARG, "NULL argument") : DDM_ERR_ARG;
  int rc = check_material(ctx, mat);
  if (rc) return rc;
  if (mode != DDM_FMM && mode != DDM_DIRECT &&
      !((mode & 0xff) == DDM_BBFMM && ((mode >> 8) & 0xff) >= 2 && ((mode >> 8) & 0xff) <= 8 &&
        (mode >> 16) == 0))
    return set_error(ctx, DDM_ERR_ARG, "bad mode");
  cudaStream_t s = (cudaStream_t)stream;
  const int ncomp = mat->kind == 1 ? 3 : 2;
  if (!ctx->exchange) return fmm_matvec(ctx, t, mat, elapsed, D, false, y, nullptr, mode, s);
  if ((rc = fmm_workspace(ctx, t, s))) return rc;   // t->y_sorted exists before it is passed
  rc = fmm_matvec(ctx, t, mat, elapsed, D, false, nullptr, t->y_sorted, mode, s);
  if (rc) return rc;
  stage_begin(ctx, DDM_ST_COMM, s);
  rc = allgather_sorted(ctx, t, t->y_sorted, ncomp, s);
  if (rc) return rc;
  stage_end(ctx, DDM_ST_COMM, s);
  scatter_user<<<nblk(t->n, 256), 256, 0, s>>>(t->n, ncomp, t->perm, t->y_sorted, y);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

// E_j = D^(h+1-j) - D^(h-j) with D^h = D^(-1) = 0   (telescoped lag kernels)
__global__ void lag_difference(int64_t len, int h, int j, const double* __restrict__ Dh,
                               double* __restrict__ E) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  const int a = h + 1 - j, b = h - j;
  const double va = (a >= 0 && a < h) ? Dh[(int64_t)a * len + i] : 0.0;
  const double vb = (b >= 0 && b < h) ? Dh[(int64_t)b * len + i] : 0.0;
  E[i] = va - vb;
}

// out = a - b (elementwise; out may alias a)
__global__ void sub_kernel(int64_t len, const double* a, const double* __restrict__ b,
                           double* out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < len) out[i] = a[i] - b[i];
}

// GMRES initial guess of step h of the march: polynomial extrapolation in
// time of D^{h-1} .. D^{h-1-q} (q = order, lowered while fewer steps exist),
// each product and sum rounded separately in the listed order
__global__ void march_guess_kernel(int64_t len, int q, const double* __restrict__ d1,
                                   const double* __restrict__ d2, const double* __restrict__ d3,
                                   const double* __restrict__ d4, const double* __restrict__ d5,
                                   const double* __restrict__ d6, double* __restrict__ x) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= len) return;
  double v;
  if (q == 5)        // 6 D1 - 15 D2 + 20 D3 - 15 D4 + 6 D5 - D6
    v = __dsub_rn(__dadd_rn(__dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(6.0, d1[i]), __dmul_rn(15.0, d2[i])),
                                                __dmul_rn(20.0, d3[i])),
                                      __dmul_rn(15.0, d4[i])),
                            __dmul_rn(6.0, d5[i])),
                  d6[i]);
  else if (q == 4)   // 5 D1 - 10 D2 + 10 D3 - 5 D4 + D5
    v = __dadd_rn(__dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(5.0, d1[i]), __dmul_rn(10.0, d2[i])),
                                      __dmul_rn(10.0, d3[i])),
                            __dmul_rn(5.0, d4[i])),
                  d5[i]);
  else if (q == 3)   // 4 D1 - 6 D2 + 4 D3 - D4
    v = __dsub_rn(__dadd_rn(__dsub_rn(__dmul_rn(4.0, d1[i]), __dmul_rn(6.0, d2[i])),
                            __dmul_rn(4.0, d3[i])), d4[i]);
  else if (q == 2)   // 3 (D1 - D2) + D3
    v = __dadd_rn(__dmul_rn(__dsub_rn(d1[i], d2[i]), 3.0), d3[i]);
  else if (q == 1)   // 2 D1 - D2
    v = __dsub_rn(__dmul_rn(d1[i], 2.0), d2[i]);
  else
    v = d1[i];
  x[i] = v;
}

__global__ void axpy_kernel(int64_t len, const double* __restrict__ x, double* __restrict__ y) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < len) y[i] += x[i];
}

// r = sum_{m=1}^{h} [K((m+1) dt) - K(m dt)] D^(h-m)
//   = sum_{j=1}^{h+1} K(j dt) (D^(h+1-j) - D^(h-j))   (D^h = D^(-1) = 0)
// i.e. h+1 continuous-source matvecs, each with its own elapsed time.
int ddm_history_apply(ddm_ctx_t ctx, ddm_tree_t t, const ddm_material* mat, double dt, int h,
                      const double* D_hist, double* r, int mode, void* stream) {
  if (!ctx || !t || !r) return ctx ? set_error(ctx, DDM_ERR_ARG, "NULL argument") : DDM_ERR_ARG;
  int rc = check_material(ctx, mat);
  if (rc) return rc;
  if (h < 0 || !(dt > 0)) return set_error(ctx, DDM_ERR_ARG, "need h >= 0 and dt > 0");
  if (mode != DDM_FMM && mode != DDM_DIRECT && mode != DDM_HIST_PERLAG)
    return set_error(ctx, DDM_ERR_ARG, "bad mode");
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t len = t->n * 3;
  DDM_CUDA(ctx, cudaMemsetAsync(r, 0, (size_t)len * sizeof(double), s));
  if (h == 0 || mat->kind == 0) return DDM_OK;   // empty sum / elastic (R10)
  if (!D_hist) return set_error(ctx, DDM_ERR_ARG, "NULL D_hist");
  if (mode == DDM_FMM) {   // fast form (f1)
    if (!ctx->exchange) return fmm_history(ctx, t, mat, dt, h, D_hist, r, nullptr, s);
    if ((rc = fmm_workspace(ctx, t, s))) return rc;   // t->y_sorted exists before it is passed
    rc = fmm_history(ctx, t, mat, dt, h, D_hist, nullptr, t->y_sorted, s);
    if (rc) return rc;
    stage_begin(ctx, DDM_ST_COMM, s);
    rc = allgather_sorted(ctx, t, t->y_sorted, 3, s);
    if (rc) return rc;
    stage_end(ctx, DDM_ST_COMM, s);
    scatter_user<<<nblk(t->n, 256), 256, 0, s>>>(t->n, 3, t->perm, t->y_sorted, r);
    DDM_CUDA(ctx, cudaGetLastError());
    return DDM_OK;
  }
  const int mv_mode = mode == DDM_DIRECT ? DDM_DIRECT : DDM_FMM;
  double* E = nullptr;
  double* y = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&E, len * sizeof(double), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&y, len * sizeof(double), s));
  for (int j = 1; j <= h + 1 && !rc; ++j) {
    lag_difference<<<nblk(len, 256), 256, 0, s>>>(len, h, j, D_hist, E);
    rc = cuda_error_if(ctx, cudaGetLastError(), "lag_difference");
    if (!rc) rc = ddm_matvec(ctx, t, mat, j * dt, E, y, mv_mode, stream);
    if (!rc) {
      axpy_kernel<<<nblk(len, 256), 256, 0, s>>>(len, y, r);
      rc = cuda_error_if(ctx, cudaGetLastError(), "axpy");
    }
  }
  cudaFreeAsync(E, s);
  cudaFreeAsync(y, s);
  return rc;
}

int ddm_history_rhs(ddm_ctx_t ctx, ddm_tree_t t, const ddm_material* mat, double dt, int h,
                    const double* D_hist, const double* b, double* rhs, int mode, void* stream) {
  if (!ctx || !t || !b || !rhs) return ctx ? set_error(ctx, DDM_ERR_ARG, "NULL argument") : DDM_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  const int64_t len = t->n * 3;
  double* r = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&r, (size_t)len * sizeof(double), s));
  int rc = ddm_history_apply(ctx, t, mat, dt, h, D_hist, r, mode, stream);
  if (!rc) {
    sub_kernel<<<nblk(len, 256), 256, 0, s>>>(len, b, r, rhs);
    rc = cuda_error_if(ctx, cudaGetLastError(), "sub_kernel");
  }
  cudaFreeAsync(r, s);
  return rc;
}

int ddm_march_guess(ddm_ctx_t ctx, int h, const double* D_hist, int64_t len, int order,
                    double* x, void* stream) {
  if (!ctx) return DDM_ERR_ARG;
  if (h < 0 || len < 0 || order < 0 || order > 5 || !x || (h > 0 && !D_hist))
    return set_error(ctx, DDM_ERR_ARG, "march_guess: bad argument");
  cudaStream_t s = (cudaStream_t)stream;
  if (len == 0) return DDM_OK;
  if (h == 0) {
    DDM_CUDA(ctx, cudaMemsetAsync(x, 0, (size_t)len * sizeof(double), s));
    return DDM_OK;
  }
  const int q = std::min(order, h - 1);
  auto prev = [&](int j) { return D_hist + (int64_t)(h - 1 - std::min(j, h - 1)) * len; };
  march_guess_kernel<<<nblk(len, 256), 256, 0, s>>>(len, q, prev(0), prev(1), prev(2), prev(3),
                                                     prev(4), prev(5), x);
  return cuda_error_if(ctx, cudaGetLastError(), "march_guess_kernel");
}

int ddm_precond_apply(ddm_ctx_t ctx, ddm_tree_t t, const ddm_material* mat, double dt,
                      const double* x, double* y, int kind, void* stream) {
  if (!ctx || !t || !x || !y) return ctx ? set_error(ctx, DDM_ERR_ARG, "NULL argument") : DDM_ERR_ARG;
  int rc = check_material(ctx, mat);
  if (rc) return rc;
  if (kind != 1 && kind != 2) return set_error(ctx, DDM_ERR_ARG, "kind must be 1 or 2");
  if (mat->kind == 1 && !(dt > 0)) return set_error(ctx, DDM_ERR_ARG, "poroelastic needs dt > 0");
  return precond_apply_user(ctx, t, mat, dt, kind, x, y, (cudaStream_t)stream);
}

int ddm_gmres_solve(ddm_ctx_t ctx, ddm_tree_t t, const ddm_material* mat, double dt,
                    const double* b, double* x, double tol, int restart, int max_iter, int mode,
                    int* iters, double* rel_resid, void* stream) {
  if (!ctx || !t || !b || !x) return ctx ? set_error(ctx, DDM_ERR_ARG, "NULL argument") : DDM_ERR_ARG;
  int rc = check_material(ctx, mat);
  if (rc) return rc;
  if (!(tol > 0) || restart < 1 || max_iter < 0)
    return set_error(ctx, DDM_ERR_ARG, "need tol > 0, restart >= 1, max_iter >= 0");
  if (mat->kind == 1 && !(dt > 0))
    return set_error(ctx, DDM_ERR_ARG, "poroelastic GMRES needs dt > 0");
  return gmres_solve(ctx, t, mat, dt, b, x, tol, restart, max_iter, mode, iters, rel_resid,
                     (cudaStream_t)stream);
}

int ddm_farfield_rhs(ddm_ctx_t ctx, const double* beta, int64_t n, int ncomp, double p_f,
                     double sH, double sh, int net, double b_p, double* b, void* stream) {
  if (!ctx || !beta || !b || n < 1 || (ncomp != 2 && ncomp != 3))
    return ctx ? set_error(ctx, DDM_ERR_ARG, "bad argument") : DDM_ERR_ARG;
  farfield_kernel<<<nblk(n, 256), 256, 0, (cudaStream_t)stream>>>(beta, n, ncomp, p_f, sH, sh,
                                                                  net, b_p, b);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int ddm_sif(ddm_ctx_t ctx, const double* w_tip, const double* ds_tip, const double* a_tip,
            int ntips, double E, double nu, double* KI, double* KII, void* stream) {
  if (!ctx || ntips < 0 || (ntips && (!w_tip || !ds_tip || !a_tip || !KI || !KII)))
    return ctx ? set_error(ctx, DDM_ERR_ARG, "bad argument") : DDM_ERR_ARG;
  if (ntips == 0) return DDM_OK;
  sif_kernel<<<nblk(ntips, 128), 128, 0, (cudaStream_t)stream>>>(w_tip, ds_tip, a_tip, ntips, E,
                                                                 nu, KI, KII);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int ddm_tip_growth(ddm_ctx_t ctx, int ntips, const double* KI, const double* KII,
                   const double* x, const double* y, const double* a, const double* beta,
                   const int* end, double K_IC, int* grow, double* new_x, double* new_y,
                   double* new_a, double* new_beta, int* new_end, void* stream) {
  if (!ctx) return DDM_ERR_ARG;
  if (ntips < 0 || !(K_IC >= 0.0) ||
      (ntips && (!KI || !KII || !x || !y || !a || !beta || !end || !grow || !new_x || !new_y ||
                 !new_a || !new_beta || !new_end)))
    return set_error(ctx, DDM_ERR_ARG, "bad argument");
  if (ntips == 0) return DDM_OK;
  tip_growth_kernel<<<nblk(ntips, 128), 128, 0, (cudaStream_t)stream>>>(
      ntips, KI, KII, x, y, a, beta, end, K_IC, grow, new_x, new_y, new_a, new_beta, new_end);
  DDM_CUDA(ctx, cudaGetLastError());
  return DDM_OK;
}

int ddm_probe_fp64(ddm_ctx_t ctx, double* tflops, void* stream) {
  if (!ctx || !tflops) return DDM_ERR_ARG;
  cudaStream_t s = (cudaStream_t)stream;
  int nsm = 148;
  cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, ctx->device);
  const int blocks = nsm * 8, threads = 256, iters = 4096;
  cudaEvent_t e0, e1;
  DDM_CUDA(ctx, cudaEventCreate(&e0));
  DDM_CUDA(ctx, cudaEventCreate(&e1));
  dfma_probe_kernel<<<blocks, threads, 0, s>>>(iters, 0.999999, 1e-7, ctx->d_scalar);  // warm-up
  float best = 1e30f;
  for (int rep = 0; rep < 5; ++rep) {
    DDM_CUDA(ctx, cudaEventRecord(e0, s));
    dfma_probe_kernel<<<blocks, threads, 0, s>>>(iters, 0.999999, 1e-7, ctx->d_scalar);
    DDM_CUDA(ctx, cudaEventRecord(e1, s));
    DDM_CUDA(ctx, cudaEventSynchronize(e1));
    float ms = 0.f;
    DDM_CUDA(ctx, cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = 2.0 * 8.0 * iters * (double)blocks * threads;
  *tflops = flops / (best * 1e-3) / 1e12;
  return DDM_OK;
}

int ddm_split_costs(const int64_t* prefix_excl, int64_t total, int nleaves, int world,
                    int* split) {
  if (!prefix_excl || !split || world < 1 || nleaves < 0) return DDM_ERR_ARG;
  split_costs(prefix_excl, total, nleaves, world, split);
  return DDM_OK;
}

}  // extern "C"
