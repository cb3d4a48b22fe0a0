// Device helpers shared by the FMM kernels (complex fp64 arithmetic, fast
// reciprocal, block copies, cell geometry) and the launcher declarations.
#pragma once
#include "ddm_internal.cuh"

namespace ddm {

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// acc += a * b
__device__ __forceinline__ void cmac(double2& acc, double2 a, double2 b) {
  acc.x = fma(a.x, b.x, fma(-a.y, b.y, acc.x));
  acc.y = fma(a.x, b.y, fma(a.y, b.x, acc.y));
}
__device__ __forceinline__ double2 cscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

// 1/x for x > 0 normal: MUFU.RCP64H seed + cubic Newton refinement (error ~e^3)
__device__ __forceinline__ double fast_rcp(double x) {
  double r;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x));
  const double e = fma(-x, r, 1.0);
  return fma(r, fma(e, e, e), r);
}

// mbarrier + 1-D TMA bulk copy (global -> shared, completion on the mbarrier)
__device__ __forceinline__ unsigned smem_u32(const void* p) {
  return (unsigned)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(unsigned bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(unsigned bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned phase) {
  asm volatile(
      "{\n .reg .pred p;\n"
      "DDM_WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      " @!p bra DDM_WAIT_%=;\n}" ::"r"(bar),
      "r"(phase)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(unsigned dst, const void* src, unsigned bytes,
                                         unsigned bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          dst),
      "l"(src), "r"(bytes), "r"(bar)
      : "memory");
}

// Block-wide global -> shared copy with 8 loads in flight per thread.
template <class T>
__device__ __forceinline__ void block_copy(T* __restrict__ dst, const T* __restrict__ src, int n) {
  const int step = blockDim.x;
  int f = threadIdx.x;
  for (; f + 7 * step < n; f += 8 * step) {
    T v[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) v[k] = src[f + k * step];
#pragma unroll
    for (int k = 0; k < 8; ++k) dst[f + k * step] = v[k];
  }
  for (; f < n; f += step) dst[f] = src[f];
}

struct CellGeom {
  double x_min, y_min, W;
  __device__ __forceinline__ double side(int lev) const { return ldexp(W, -lev); }
  __device__ __forceinline__ double2 centre(int lev, int ix, int iy) const {
    const double s = ldexp(W, -lev);
    return make_double2(x_min + (ix + 0.5) * s, y_min + (iy + 0.5) * s);
  }
};

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

// Biot constants of a poroelastic material at elapsed time tau (poro.cu)
struct PoroParams {
  double G = 0, C = 0, eta = 0, kp = 0, S = 0, kappa = 0, c = 0, ct = 0;
};
PoroParams poro_params(const ddm_material* m, double tau);
int poro_init_tables(ddm_ctx_s* ctx);

// far-field (expansion) weights of the poroelastic kernel, r >> sqrt(c tau)
// (DESIGN.md §4.5): Phi scaled by fu = 1 + 2 eta k_p = (1-nu)/(1-nu_u); Psi~
// gains the monopole / fluid-source I2 terms and the c tau I4 term; L2P reads
// p = -4 k_p Re(Phi_total)/fu (formula sign; ABI p = -that).
// lin = 1: only the part proportional to c tau (the far form is affine in
// tau: F(tau) = F0 + tau F1) -- the far field of the fast history sum, whose
// tau-independent part cancels (sum_j E_j = 0).
struct PoroFar {
  int on = 0, lin = 0;
  double fu = 1.0, eta = 0, kp = 0, S = 0, kappa = 0, ct = 0, gc = 1.0;
};
inline PoroFar poro_far(const PoroParams& P) {
  PoroFar f;
  f.on = 1;
  f.fu = 1.0 + 2.0 * P.eta * P.kp;
  f.eta = P.eta; f.kp = P.kp; f.S = P.S; f.kappa = P.kappa; f.ct = P.ct; f.gc = P.G * P.C;
  return f;
}

int launch_poro_prep(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D,
                     cudaStream_t s);
int launch_poro_p2p(ddm_ctx_s* ctx, ddm_tree_s* t, int item_lo, int item_hi, const PoroParams& P,
                    cudaStream_t s);
// near-field matrix cache of the poroelastic operator (built on the second
// consecutive matvec with the same parameters)
int poro_near_cache_update(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, cudaStream_t s);
// history lag cache: true when lags 1..h+1 are cached
bool poro_hist_cache_update(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                            int h, cudaStream_t s, int* rc_out);
int launch_poro_hist_cached(ddm_ctx_s* ctx, ddm_tree_s* t, int h, const double* Hs,
                            cudaStream_t s);
int launch_poro_hist_gather(ddm_ctx_s* ctx, ddm_tree_s* t, int h, const double* D_hist,
                            double* Hs, double* Cs, double* Ctot, cudaStream_t s);
int launch_poro_hist_near(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, int h, double dt,
                          const double* Hs, const double* Cs, cudaStream_t s);
int launch_poro_self_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, double* blk,
                            cudaStream_t s);
// leaf-block Jacobi preconditioner blocks (gmres.cu): chunks[q] = (first
// sorted element, count <= kPcChunk), block q row-major at blk + off[q]
int launch_poro_chunk_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, const PoroParams& P, int nchunks,
                             const int2* chunks, const int64_t* off, double* blk, cudaStream_t s);
int launch_elastic_chunk_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, double gc, int nchunks,
                                const int2* chunks, const int64_t* off, double* blk,
                                cudaStream_t s);
int launch_elastic_self_blocks(ddm_ctx_s* ctx, ddm_tree_s* t, double gc, double* blk,
                               cudaStream_t s);
int launch_poro_direct(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi,
                       const PoroParams& P, double* y_user, double* y_sorted, cudaStream_t s);

// ---- launchers (expansions.cu): upward / downward passes
struct PoroFar;
// scope 0: P2M of all leaves + M2M of every non-leaf cell (replicated);
// 1: P2M of the owned leaves + M2M of this rank's complete cells; 2: M2M of
// the straddling cells (after the multipole exchange)
enum { kUpFull = 0, kUpOwn = 1, kUpStrad = 2 };
int launch_upward(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D, int ncomp,
                  const PoroFar& pf, cudaStream_t s, int scope = kUpFull);
// multipoles of this rank's complete cells -> t->xsend; gathered -> mpole
int launch_mpole_pack(ddm_ctx_s* ctx, ddm_tree_s* t, int rank, cudaStream_t s);
int launch_mpole_unpack(ddm_ctx_s* ctx, ddm_tree_s* t, int rank, int world, cudaStream_t s);
// use_x: the M2L adds the P2L series (local_x) of the leaves with X lists
int launch_downward(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s, bool use_x = false);
int launch_l2p(ddm_ctx_s* ctx, ddm_tree_s* t, int ncomp, double gc, const PoroFar& pf,
               cudaStream_t s);
// P2L of the owned leaves' X lists into t->local_x, elastic
int launch_p2l(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D, int ncomp,
               cudaStream_t s);
// static tables of the block-staged L2P (geometry of leaves / W entries, runs
// of the owned range); idempotent, outside any capture
int l2p_prepare(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s);
int launch_finalize(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, int ncomp, double gc,
                    const PoroFar& pf, double* y_user, double* y_sorted, cudaStream_t s);

// ---- launchers (p2p.cu): near field
int launch_prep_sources(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D,
                        int ncomp, cudaStream_t s);
int launch_p2p(ddm_ctx_s* ctx, ddm_tree_s* t, int item_lo, int item_hi, double gc,
               cudaStream_t s);
// leaf-block near field (records staged in shared memory by bulk copies) into
// t->y_near, and the matching assembly y = y_near + y_far; DDM_P2P_LEAF=0
// selects the item kernel (launch_p2p + launch_finalize) instead
bool use_leaf_p2p();
int launch_p2p_leaf(ddm_ctx_s* ctx, ddm_tree_s* t, double gc, cudaStream_t s, bool use_x = false);
int launch_finalize_near(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, double* y_user,
                         double* y_sorted, cudaStream_t s);
// near-field source stream (p2p.cu): chain order + break records once per
// tree; prep_stream writes the element records (and D in sorted order)
int build_source_stream(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s);
// halo: only the slots the owned leaves read (sharded multi-rank matvec)
int launch_prep_stream(ddm_ctx_s* ctx, ddm_tree_s* t, const int* perm_in, const double* D,
                       int ncomp, cudaStream_t s, bool halo = false);
int launch_direct(ddm_ctx_s* ctx, ddm_tree_s* t, int64_t lo, int64_t hi, int ncomp, double gc,
                  double* y_user, double* y_sorted, cudaStream_t s);

}  // namespace ddm
