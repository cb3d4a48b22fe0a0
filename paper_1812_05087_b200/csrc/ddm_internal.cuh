// Internal declarations of libddm (not part of the C-ABI).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <cstdlib>

#include <string>
#include <vector>

#include "../../include/ddm.h"

#ifdef DDM_WITH_NCCL
#include <nccl.h>
#endif

namespace ddm {

constexpr int kLBits = 30;      // quantisation bits per axis (R8)
constexpr int kMaxP = 40;       // max complex coefficients per series
constexpr int kNOffsets = 49;   // (dx,dy) in [-3,3]^2, class id (dy+3)*7+(dx+3)
#ifndef DDM_TGT_GROUP
#define DDM_TGT_GROUP 16
#endif
constexpr int kTgtGroup = DDM_TGT_GROUP;   // targets per P2P work item (one warp)
#ifndef DDM_SRC_CHUNK
#define DDM_SRC_CHUNK 512
#endif
constexpr int kSrcChunk = DDM_SRC_CHUNK;  // max sources per P2P work item
constexpr int kSrcStride = 12;  // doubles per direct-mode source record
// near-field stream record (p2p.cu): node + 5 complex coefficients
// {node, 2 P1, 2 P2, B/2, Q', K} (DDM_REC_K = 1, the default), or the round-1
// 10-double form {node, P1, P2, B/2, Q'} that rebuilds 2 (z - zc) from the
// carried node offsets (DDM_REC_K = 0)
#ifndef DDM_REC_K
#define DDM_REC_K 1
#endif
constexpr int kRecStride = DDM_REC_K ? 12 : 10;  // doubles per record
constexpr int kChainMax = 256;  // leaves with more elements keep Morton order (no node sharing)
#ifndef DDM_PC_CHUNK
#define DDM_PC_CHUNK 32
#endif
constexpr int kPcChunk = DDM_PC_CHUNK;   // max elements per leaf-block preconditioner block

struct Status {
  int code = DDM_OK;
  std::string msg;
};

// Per-stage CUDA events (optional profiling)
struct StageEvents {
  cudaEvent_t ev[2 * DDM_NSTAGES] = {};
  bool created = false;
};

}  // namespace ddm

struct ddm_ctx_s {
  int device = 0;
  int rank = 0, world = 1;
  // owned rows are exchanged with NCCL (world > 1, or DDM_FORCE_NCCL=1 on one
  // rank: the exchange path run on a one-rank communicator, for tests)
  bool exchange = false;
  std::string err;
  bool profiling = false;
  ddm::StageEvents stage;
  double stage_ms[DDM_NSTAGES] = {};
#ifdef DDM_WITH_NCCL
  ncclComm_t comm = nullptr;
#endif
  // fork/join streams: the far-field chain (latency bound) runs on s_hi, the
  // near field (P2P, throughput bound) concurrently on s_lo
  cudaStream_t s_hi = nullptr, s_lo = nullptr;
  cudaStream_t s_cap = nullptr;   // capture stream of the matvec graphs (fmm.cu)
  bool serial = false;            // DDM_SERIAL=1: everything on the caller's stream (profiling)
  bool serial_env = false;        // the DDM_SERIAL setting (restored when profiling mode 2 ends)
  cudaEvent_t ev_fork = nullptr, ev_far = nullptr, ev_near = nullptr, ev_p2l = nullptr;
  // persistent scratch
  double* d_scalar = nullptr;     // small device scratch (reductions)
  double* h_pinned = nullptr;     // small pinned host scratch
  size_t h_pinned_n = 0;
};

// Device-side tree and all per-geometry buffers.  Level-major cell numbering,
// Morton order within a level.
// arguments that determine a matvec's launch sequence (graph cache key)
struct MatvecKey {
  const double* D = nullptr;
  double* y_user = nullptr;
  double* y_sorted = nullptr;
  cudaStream_t s = nullptr;
  int mode = -1;
  bool d_sorted = false, serial = false;
  ddm_material mat = {};
  double elapsed = 0.0;
  bool operator==(const MatvecKey& o) const {
    return D == o.D && y_user == o.y_user && y_sorted == o.y_sorted && s == o.s &&
           mode == o.mode && d_sorted == o.d_sorted && serial == o.serial &&
           mat.kind == o.mat.kind && mat.G == o.mat.G && mat.nu == o.mat.nu &&
           mat.nu_u == o.mat.nu_u && mat.alpha == o.mat.alpha && mat.kappa == o.mat.kappa &&
           elapsed == o.elapsed;
  }
};
struct MatvecGraph {
  MatvecKey key;
  cudaGraphExec_t exec = nullptr;
};

struct ddm_tree_s {
  ddm_ctx_s* ctx = nullptr;
  double build_ms[DDM_TB_N] = {};   // ddm_tree_build_times
  int64_t n = 0;
  int leaf = 0, p = 0;
  int nlevels = 0;           // number of levels (max level + 1)
  int ncells = 0, nleaves = 0;
  int64_t nv = 0, nu = 0, near_pairs = 0;
  int nitems = 0;
  double x_min = 0, y_min = 0, W = 1;
  double a_max = 0;              // largest element half-length
  std::vector<int> level_off;    // [nlevels+1] first cell of each level
  // owned part (multi-GPU): contiguous sorted element range and leaf range
  int own_leaf_lo = 0, own_leaf_hi = 0;
  int64_t own_el_lo = 0, own_el_hi = 0;
  std::vector<int64_t> rank_el_lo;   // [world+1] sorted-element split points
  std::vector<int> rank_leaf_lo;     // [world+1] leaf split points
  std::vector<int64_t> leaf_cost_prefix;  // [nleaves+1] exclusive prefix of leaf costs

  // element data (sorted / Morton order)
  uint64_t* keys_user = nullptr;  // [n] keys in user order
  uint64_t* keys = nullptr;       // [n] sorted keys
  int* perm = nullptr;            // [n] sorted -> user
  double* ex = nullptr;           // [n] centre x
  double* ey = nullptr;           // [n] centre y
  double* ea = nullptr;           // [n] half length
  double* ec = nullptr;           // [n] cos beta
  double* es = nullptr;           // [n] sin beta
  int* el_leaf = nullptr;         // [n] leaf (position in leaf list) of each element

  // cells
  int* c_level = nullptr;
  int* c_ix = nullptr;
  int* c_iy = nullptr;
  int* c_start = nullptr;
  int* c_count = nullptr;
  int* c_parent = nullptr;
  int* c_first_child = nullptr;
  int* c_nchild = nullptr;
  int* c_leaf = nullptr;
  int* colleagues = nullptr;      // [ncells][9], -1 padded
  int* v_off = nullptr;           // [ncells+1]
  int* v_idx = nullptr;           // [nv]
  unsigned char* v_cls = nullptr; // [nv] offset class
  int* leaves = nullptr;          // [nleaves] cell ids
  int* u_off = nullptr;           // [nleaves+1]
  int* u_lo = nullptr;            // [nu]
  int* u_hi = nullptr;            // [nu]
  int* w_off = nullptr;           // [nleaves+1] W lists (M2P cells) of each leaf
  int* w_idx = nullptr;           // [nw] canonical cell ids, ascending per leaf
  int64_t nw = 0;
  int w_min = 24;                 // W(B) cells hold >= w_min elements (DDM_W_MIN, 0 = off)
  // X lists (P2L, the dual of W): per target leaf B with
  // count(B) >= x_min, the coarser leaves of U(B) that do not touch B; their
  // elements are expanded into B's local series (p2l_kernel) by the elastic
  // series FMM, whose near field then reads the U ranges minus X (ux_*).
  // Every other path (poroelastic, bbFMM, history, direct) keeps U whole.
  int xl_min = 0;                 // DDM_X_MIN at build time, 0 = off (the default: DESIGN §4.13)
  int* x_off = nullptr;           // [nleaves+1]
  int* x_idx = nullptr;           // [nx] X leaves (cell ids), ascending element start
  int64_t nx = 0;
  int* ux_off = nullptr;          // [nleaves+1] U minus X: merged element ranges per leaf
  int* ux_lo = nullptr;           // [nux]
  int* ux_hi = nullptr;           // [nux]
  int64_t nux = 0, near_pairs_x = 0;   // ranges, and the P2P pairs of U minus X
  int2* lr_rng_x = nullptr;       // [nux] record ranges of the ux ranges
  int4* leaf_info_x = nullptr;    // [nleaves] (c_start, c_count, ux_off[k], ux_off[k+1])
  double2* local_x = nullptr;     // [nleaves][2p] P2L local series of the leaves with X
  int* x_slot = nullptr;          // [ncells] leaf index k of a leaf with an X list, else -1
  int4* items = nullptr;          // P2P work items: (leaf, tgt0, src_begin, src_end)
  int* item_off = nullptr;        // [nleaves+1] first item of each leaf
  int item_lo_owned = 0, item_hi_owned = 0;   // P2P items of owned leaves
  int* p2p_order = nullptr;       // [item_hi_owned - item_lo_owned] owned items, most sources
                                  // first (longest-processing-time order: no tail)
  // upward-pass schedule (expansions.cu)
  // subtree passes (small trees, expansions.cu): split level, roots = its cells,
  // per (root, level >= Ls) ranges into up_list (M2M) and into the level's cells (L2L)
  int sub_Ls = 0, sub_n = 0, sub_nsl = 0;
  int2* sub_up = nullptr;
  int2* sub_cells = nullptr;
  int* up_list = nullptr;         // non-leaf cells of level >= 2, deepest level first
  int n_up = 0;
  std::vector<int> up_level_off;  // [2 (nlevels+1)]: level l = up_list[off[2l], off[2l+1])
  std::vector<int> h_up;          // host copy of up_list
  // sharded upward pass (several ranks): a cell is COMPLETE on
  // rank r when its element range lies inside r's range; r computes P2M of
  // its leaves and M2M of its complete cells, the packed multipoles of every
  // rank's complete cells are all-gathered, and the STRADDLING cells (ranges
  // across a rank boundary: ancestors of the boundaries) are completed on
  // every rank by M2M from the gathered children.
  bool shard_up = false;          // partition has several ranks
  int64_t halo_lo = 0, halo_hi = 0;   // hull of the stream slots the owned leaves read
  int2* halo_rng = nullptr;           // those slots as merged ranges [a, b) (sharded prep)
  int64_t* halo_pre = nullptr;        // [nhalo + 1] exclusive prefix of the range lengths
  int nhalo = 0;
  int64_t halo_slots = 0;
  int* xr_cells = nullptr;        // complete cells of every rank, rank-major, ascending
  std::vector<int> xr_off;        // [world+1]
  int* xr_off_dev = nullptr;      // device copy of xr_off
  int xr_max = 0;                 // max complete cells of one rank
  int* up_own = nullptr;          // this rank's complete non-leaf cells (level >= 2), deepest level first
  std::vector<int> up_own_off;    // [2 (nlevels+1)] as up_level_off
  int* dn_own = nullptr;          // cells of level >= 2 holding owned targets (ascending = level-major)
  std::vector<int> dn_own_off;    // [nlevels+1] first entry of each level (M2L / L2L lists)
  int* up_strad = nullptr;        // straddling non-leaf cells (level >= 2), deepest level first
  std::vector<int> up_strad_off;
  double2* xsend = nullptr;       // [xr_max][2p] packed multipoles of this rank
  double2* xrecv = nullptr;       // [world][xr_max][2p] gathered
  // persistent buffers of the all-gather of the owned output rows
  double* ag_send = nullptr;
  double* ag_recv = nullptr;
  int64_t* ag_lo = nullptr;       // device copy of rank_el_lo
  int64_t ag_max = 0;             // max owned rows of one rank

  // FMM operators (device, fmm.cu fmm_init_operators): every translation is
  // pre-scale (complex powers) x real Pascal matrix x post-scale
  double* op_pas = nullptr;       // [p][p]    C(m,k) at m*p+k      (L2L, lane k)
  double* op_pasT = nullptr;      // [p][p]    C(m,n) at n*p+m      (M2M, lane m)
  double* op_pm2l = nullptr;      // [p+1][p]  C(m+n,n) at n*p+m    (M2L, runtime-p path)
  double2* op_w = nullptr;        // [49][p+2] w^k, w = 1/delta      (M2L offset classes)
  double2* op_eps = nullptr;      // [4][p+2]  eps_q^k               (M2M / L2L quadrants)
  double2* op_e2i = nullptr;      // [4][p+2]  (2 eps_q)^-k
  // expansions: [ncells][2][p] complex
  double2* mpole = nullptr;
  double2* local = nullptr;
  // per-matvec workspaces
  double* src = nullptr;          // [n][12] direct-mode source records
  // near-field source stream (p2p.cu): each leaf's elements
  // reordered along fracture chains; consecutive elements sharing a node
  // share its reciprocal.  Built once per tree.
  int* st_elem = nullptr;         // [n] stream slot -> sorted element (permutation within leaves)
  unsigned char* st_code = nullptr;   // [n] bit 0: flipped (first node = z2), bit 1: linked to slot - 1
  int* rbeg = nullptr;            // [n+1] first record of each slot (its break record if unlinked)
  double* srec = nullptr;         // [nrec][kRecStride]; record 0 = pad
  int64_t nrec = 0;
  int* it_roff = nullptr;         // [nitems+1] first record range of each P2P item
  int2* it_rng = nullptr;         // record ranges [rb, re) of each item's source window
  int2* lr_rng = nullptr;         // [nu] record range [rbeg[u_lo], rbeg[u_hi]) of every U range
                                  // (leaf k's ranges: u_off[k] .. u_off[k+1]; p2p_leaf_kernel)
  int4* leaf_info = nullptr;      // [nleaves] (c_start, c_count, u_off[k], u_off[k+1]) of each leaf
  // block-staged L2P (expansions.cu): static geometry tables and the runs of
  // 128 owned elements (first leaf, leaves, first W entry, W entries)
  double4* leaf_geo = nullptr;    // [nleaves] (z0.x, z0.y, 1/s, has a local expansion)
  double4* w_geo = nullptr;       // [nw] (z_D.x, z_D.y, 1/s_D, 0) of every W entry
  int2* p2m_runs = nullptr;       // P2M runs (first leaf, leaves) over all leaves
  int2* p2m_runs_own = nullptr;   // ... over the owned leaves
  int p2m_nruns = 0, p2m_nruns_own = 0;
  int p2m_own_lo = -1, p2m_own_hi = -1;
  int4* l2p_runs = nullptr;
  int* l2p_order = nullptr;
  int* p2p_leaf_order = nullptr;  // near-field leaf launch order (owned-relative), or null       // L2P run launch order (longest first), or null
  int l2p_nruns = 0;
  int64_t l2p_lo = -1, l2p_hi = -1;   // owned range the runs were built for
  double* y_near = nullptr;       // [n][2] elastic near field of the owned elements (sorted order)
  double* gpart = nullptr;        // per-group partials of the on-the-fly poroelastic near field
  int64_t gpart_n = 0;
  double2* part = nullptr;        // [nitems*32] partial tractions
  double* d_sorted = nullptr;     // [n*3] D gathered into sorted order
  double* y_sorted = nullptr;     // [n*3]
  double* y_far = nullptr;        // [n*3] L2P far field of the owned elements (sorted order)
  // bbFMM far field (bbfmm.cu): node weights W and node values F, [ncells][3][bb_n^2] complex
  double2* bb_w = nullptr;
  double2* bb_f = nullptr;
  int bb_n = 0;
  // poroelastic near-field matrix cache (poro.cu): 3x3
  // blocks of every owned near pair for one (material, elapsed time), built
  // on the second consecutive matvec with the same parameters
  double* nc = nullptr;           // blocks, item by item: [(jpos * kTgtGroup + t) * 9 + 3 r + c]
  int64_t* nc_off = nullptr;      // [owned items] first double of each item
  int64_t nc_n = 0;               // doubles allocated
  double nc_key[9] = {};          // PoroConst of the cached blocks
  double nc_seen[9] = {};         // PoroConst of the previous poroelastic matvec
  bool nc_valid = false, nc_seen_set = false;
  // history near-field lag cache (poro.cu): blocks of the
  // poroelastic part K^p(j dt) of every owned near pair, in chunks of lags
  // (nc_off item layout x kLagChunk), built as the history grows
  std::vector<double*> hc_lag;    // device chunks of kLagChunk lags ([item][jpos][lag][t][9])
  std::vector<double*> hc_alloc;  // the allocations holding them (doubling groups of chunks)
  int hc_nlags = 0;               // lags built (1..hc_nlags)
  int hc_max_chunks = 0;          // chunk budget (memory) fixed when the cache is keyed
  double** hc_ptrs = nullptr;     // device copy of hc_lag
  int hc_ptrs_n = 0;
  double hc_key[9] = {}, hc_seen[9] = {};
  bool hc_valid = false, hc_seen_set = false, hc_capped = false;
  // matvec CUDA graphs (fmm.cu)
  std::vector<MatvecGraph> graphs = std::vector<MatvecGraph>(4);
  int graph_next = 0;
  MatvecKey seen_keys[4];          // recently used argument sets (capture on a repeat)
  int seen_next = 0;
  // GMRES block-Jacobi preconditioner: inverse self blocks [n][ncomp][ncomp]
  // (sorted order) for the material / elapsed time in pc_key
  double* pc = nullptr;
  double pc_key[8] = {};
  // leaf-block Jacobi (default GMRES preconditioner): chunks of <= kPcChunk
  // consecutive sorted elements of one leaf, inverse blocks column-major
  int2* pc_chunks = nullptr;      // [pc_nchunks] (first sorted element, count)
  int64_t* pc_off = nullptr;      // [pc_nchunks] block offsets (doubles), for ncomp = pc_off_ncomp
  int pc_nchunks = 0, pc_off_ncomp = 0;
  int pc_q_lo = 0, pc_q_hi = 0;   // chunks of the owned elements
  double* pcl = nullptr;
  int64_t pcl_n = 0;
  double pcl_key[8] = {};
  // GMRES workspace
  double* krylov = nullptr;
  int krylov_m = 0;
  int64_t krylov_dof = 0;
  double* gm_w = nullptr;
  double* gm_tmp = nullptr;
  double* gm_part = nullptr;
  int64_t gm_part_n = 0;
  // device Arnoldi state of the batched GMRES (gmres.cu): packed Hessenberg,
  // Givens rotations, rotated rhs, per-step estimates, 1/h(k+1,k), flags
  double* gm_dev = nullptr;
  int gm_dev_m = 0;
  unsigned* gm_ticket = nullptr;  // zeroed tickets of the fused GMRES reductions
  int gm_ticket_n = 0;
  // captured Arnoldi step (gmres.cu): one graph per argument set
  cudaGraphExec_t gm_exec = nullptr;
  double* gm_pin = nullptr;       // pinned host: GMRES residual estimates + breakdown flag
  int gm_pin_n = 0;
  uintptr_t gm_key[12] = {};
};

namespace ddm {

// error helpers (api.cu)
int set_error(ddm_ctx_s* ctx, int code, const std::string& msg);
int cuda_error(ddm_ctx_s* ctx, cudaError_t e, const char* what);
int cuda_error_if(ddm_ctx_s* ctx, cudaError_t e, const char* what);

#define DDM_CUDA(ctx, call)                                             \
  do {                                                                  \
    cudaError_t e_ = (call);                                            \
    if (e_ != cudaSuccess) return ::ddm::cuda_error((ctx), e_, #call);  \
  } while (0)

#define DDM_CHECK_LAUNCH(ctx, name) DDM_CUDA(ctx, cudaGetLastError())

// DDM_POISON=1 (tests; compute-sanitizer is not available on the GPU pool):
// every library allocation is filled with 0xFF bytes (NaN doubles, -1
// indices), so a kernel that reads memory no kernel wrote shows up as NaN in
// a checked result (or as a fault)
inline bool poison_allocs() {
  static const bool on = [] {
    const char* v = getenv("DDM_POISON");
    return v && v[0] == '1';
  }();
  return on;
}

template <class T>
int dalloc(ddm_ctx_s* ctx, T** p, size_t count) {
  *p = nullptr;
  if (count == 0) count = 1;
  cudaError_t e = cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, DDM_ERR_OOM, std::string("cudaMalloc failed: ") + cudaGetErrorString(e));
  }
  if (poison_allocs()) cudaMemset(*p, 0xff, count * sizeof(T));
  return DDM_OK;
}

// Tree-lifetime allocation from the stream-ordered pool (the context keeps
// the pool's memory mapped): no device-wide synchronisation per array, unlike
// cudaMalloc.  Freed by free_tree with cudaFree (valid for pool memory).
template <class T>
int talloc(ddm_ctx_s* ctx, T** p, size_t count, cudaStream_t s) {
  *p = nullptr;
  if (count == 0) count = 1;
  static const bool pool = [] {
    const char* v = getenv("DDM_TREE_POOL");
    return !(v && v[0] == '0');
  }();
  cudaError_t e = pool ? cudaMallocAsync((void**)p, count * sizeof(T), s)
                       : cudaMalloc((void**)p, count * sizeof(T));
  if (e != cudaSuccess) {
    cudaGetLastError();
    return set_error(ctx, DDM_ERR_OOM, std::string("cudaMallocAsync failed: ") + cudaGetErrorString(e));
  }
  if (poison_allocs()) cudaMemsetAsync(*p, 0xff, count * sizeof(T), s);
  return DDM_OK;
}

// scan.cu
int exclusive_scan_i32(ddm_ctx_s* ctx, const int* in, int* out, int n, int* total_host,
                       cudaStream_t s);
int exclusive_scan_i64(ddm_ctx_s* ctx, const int64_t* in, int64_t* out, int n, int64_t* total_host,
                       cudaStream_t s);

// tree.cu
int build_tree(ddm_ctx_s* ctx, const double* xc, const double* yc, const double* a,
               const double* beta, int64_t n, int leaf, int p, double min_side,
               cudaStream_t s, ddm_tree_s* t);
void free_tree(ddm_tree_s* t);
int partition_tree(ddm_tree_s* t, int rank, int world, cudaStream_t s);
void shard_owner(const int* c_start, const int* c_count, int ncells, const int64_t* lo, int world,
                 int* owner);
void split_costs(const int64_t* prefix_excl, int64_t total, int nleaves, int world, int* split);

// fmm.cu
int fmm_init_operators(ddm_tree_s* t, cudaStream_t s);
// Destroy every captured matvec graph and forget the recently seen argument
// sets.  Called whenever a buffer a captured graph may read or write is
// rebuilt or reallocated (poroelastic near-field cache, bbFMM node arrays,
// group partials, partition change): a graph holds raw pointers and would
// otherwise replay against stale or freed memory.
void drop_graphs(ddm_tree_s* t);
// D: [n][ncomp], user order (d_sorted = false) or sorted order (true), full
// length.  Writes the owned rows into y_user (user order, via perm) and/or
// y_sorted.  ncomp = 2 (elastic) or 3 (poroelastic, elapsed = tau).
int fmm_workspace(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s);
int fmm_matvec(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double elapsed,
               const double* D, bool d_sorted, double* y_user, double* y_sorted, int mode,
               cudaStream_t s);

// several ranks emulated on one device (fmm.cu; tests)
int fmm_matvec_sim(ddm_ctx_s* ctx, ddm_tree_s* const* trees, int world, const ddm_material* mat,
                   const double* D, double* y, cudaStream_t s);
int launch_scatter_user(ddm_ctx_s* ctx, ddm_tree_s* t, const double* ys, int ncomp, double* y,
                        cudaStream_t s);

// fast history sum (poroelastic): r = sum_{m=1}^{h} A^(m) D^(h-m), D_hist user order
int fmm_history(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt, int h,
                const double* D_hist, double* y_user, double* y_sorted, cudaStream_t s);

// bbfmm.cu: Chebyshev far field with n nodes per dimension (mode DDM_BBFMM)
int bb_prepare(ddm_ctx_s* ctx, ddm_tree_s* t, int n);
int launch_bb_far(ddm_ctx_s* ctx, ddm_tree_s* t, int n, const double* D, int ncomp, double gc,
                  cudaStream_t s);

// gmres.cu
int gmres_solve(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                const double* b, double* x, double tol, int restart, int max_iter, int mode,
                int* iters, double* rel_resid, cudaStream_t s);

// y = M^-1 x (user order): kind 1 point-block, 2 leaf-block Jacobi
int precond_apply_user(ddm_ctx_s* ctx, ddm_tree_s* t, const ddm_material* mat, double dt,
                       int kind, const double* x_user, double* y_user, cudaStream_t s);

// comm (api.cu)
int allgather_sorted(ddm_ctx_s* ctx, ddm_tree_s* t, double* buf, int ncomp, cudaStream_t s);
int allgather_mpole(ddm_ctx_s* ctx, ddm_tree_s* t, cudaStream_t s);
int allreduce_sum(ddm_ctx_s* ctx, double* buf, int64_t count, cudaStream_t s);

// profiling helpers
void stage_begin(ddm_ctx_s* ctx, int st, cudaStream_t s);
void stage_end(ddm_ctx_s* ctx, int st, cudaStream_t s);

}  // namespace ddm
