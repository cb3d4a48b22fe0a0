// Tree build on the GPU (§3.1):
//   a1 Morton keys: quantise centres into the root square, bit-interleave
//      (x in bit 0 -> child slot 1 + xbit + 2 ybit, the paper's left->right,
//      bottom->top indexing);
//   a2 stable LSD radix sort of (key, user index), 8 bits per pass;
//   a3 cells level by level from sorted keys: a cell exists iff non-empty and
//      its parent holds more than `leaf` elements;
//   a4 colleague (same-level neighbour) lists, V lists ("not neighbors at the
//      same level, but their parents are neighbors") and U lists
//      (near field, as merged source-element ranges) + P2P work items.
#include <algorithm>
#include <cmath>
#include <cstring>

#include "ddm_internal.cuh"

namespace ddm {
namespace {

constexpr int kRadixThreads = 256;
constexpr int kRadixItems = 16;
constexpr int kRadixTile = kRadixThreads * kRadixItems;

__device__ __forceinline__ uint64_t spread_bits(uint32_t v) {
  uint64_t x = v & 0x3fffffffu;
  x = (x | (x << 16)) & 0x0000FFFF0000FFFFull;
  x = (x | (x << 8)) & 0x00FF00FF00FF00FFull;
  x = (x | (x << 4)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x << 2)) & 0x3333333333333333ull;
  x = (x | (x << 1)) & 0x5555555555555555ull;
  return x;
}

__device__ __forceinline__ uint32_t compact_bits(uint64_t x) {
  x &= 0x5555555555555555ull;
  x = (x | (x >> 1)) & 0x3333333333333333ull;
  x = (x | (x >> 2)) & 0x0F0F0F0F0F0F0F0Full;
  x = (x | (x >> 4)) & 0x00FF00FF00FF00FFull;
  x = (x | (x >> 8)) & 0x0000FFFF0000FFFFull;
  x = (x | (x >> 16)) & 0x00000000FFFFFFFFull;
  return (uint32_t)x;
}

// ---------------------------------------------------------------- a1
// Root square and input validation in one pass (a1): per block the min/max
// of the centres and the largest half-length; bad |= 1 for a non-finite
// centre, 2 for a half-length that is not finite and > 0.
__global__ void minmax_partial(const double* __restrict__ x, const double* __restrict__ y,
                               const double* __restrict__ ha, int64_t n,
                               double4* __restrict__ part, double* __restrict__ pamax,
                               int* __restrict__ bad) {
  double xmn = INFINITY, xmx = -INFINITY, ymn = INFINITY, ymx = -INFINITY, am = 0.0;
  int flags = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const double a = x[i], b = y[i], h = ha[i];
    if (!isfinite(a) || !isfinite(b)) flags |= 1;
    if (!(isfinite(h) && h > 0.0)) flags |= 2;
    xmn = fmin(xmn, a); xmx = fmax(xmx, a); ymn = fmin(ymn, b); ymx = fmax(ymx, b);
    am = fmax(am, h);
  }
  for (int o = 16; o; o >>= 1) {
    xmn = fmin(xmn, __shfl_xor_sync(0xffffffffu, xmn, o));
    xmx = fmax(xmx, __shfl_xor_sync(0xffffffffu, xmx, o));
    ymn = fmin(ymn, __shfl_xor_sync(0xffffffffu, ymn, o));
    ymx = fmax(ymx, __shfl_xor_sync(0xffffffffu, ymx, o));
    am = fmax(am, __shfl_xor_sync(0xffffffffu, am, o));
  }
  __shared__ double4 sh[32];
  __shared__ double sa[32];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) {
    sh[w] = make_double4(xmn, xmx, ymn, ymx);
    sa[w] = am;
  }
  if (flags) atomicOr(bad, flags);
  __syncthreads();
  if (threadIdx.x == 0) {
    double4 r = sh[0];
    double ra = sa[0];
    for (int k = 1; k < (int)(blockDim.x >> 5); ++k) {
      r.x = fmin(r.x, sh[k].x); r.y = fmax(r.y, sh[k].y);
      r.z = fmin(r.z, sh[k].z); r.w = fmax(r.w, sh[k].w);
      ra = fmax(ra, sa[k]);
    }
    part[blockIdx.x] = r;
    pamax[blockIdx.x] = ra;
  }
}

__global__ void morton_kernel(const double* __restrict__ x, const double* __restrict__ y,
                              int64_t n, double xmin, double ymin, double s,
                              uint64_t* __restrict__ key, int* __restrict__ idx) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double top = (double)((1u << kLBits) - 1);
  // one IEEE subtract, then one IEEE multiply, never fused (reading R8)
  double fx = floor(__dmul_rn(__dsub_rn(x[i], xmin), s));
  double fy = floor(__dmul_rn(__dsub_rn(y[i], ymin), s));
  fx = fmin(fmax(fx, 0.0), top);
  fy = fmin(fmax(fy, 0.0), top);
  key[i] = spread_bits((uint32_t)fx) | (spread_bits((uint32_t)fy) << 1);
  idx[i] = (int)i;
}

// ---------------------------------------------------------------- a2
__global__ void radix_hist(const uint64_t* __restrict__ k, int64_t n, int shift,
                           int* __restrict__ hist, int nblocks) {
  __shared__ int h[256];
  h[threadIdx.x] = 0;
  __syncthreads();
  const int64_t t0 = (int64_t)blockIdx.x * kRadixTile;
  for (int r = 0; r < kRadixItems; ++r) {
    const int64_t i = t0 + r * kRadixThreads + threadIdx.x;
    if (i < n) atomicAdd(&h[(k[i] >> shift) & 255], 1);
  }
  __syncthreads();
  hist[threadIdx.x * nblocks + blockIdx.x] = h[threadIdx.x];
}

// Stable scatter: items of a tile are visited in order (round r, warp w, lane).
__global__ void radix_scatter(const uint64_t* __restrict__ kin, const int* __restrict__ vin,
                              uint64_t* __restrict__ kout, int* __restrict__ vout, int64_t n,
                              int shift, const int* __restrict__ offs, int nblocks) {
  __shared__ int base[256];
  __shared__ int wcnt[kRadixThreads / 32][256];
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  base[tid] = offs[tid * nblocks + blockIdx.x];
  const unsigned lt = (1u << lane) - 1u;
  const int64_t t0 = (int64_t)blockIdx.x * kRadixTile;
  for (int r = 0; r < kRadixItems; ++r) {
    const int64_t i = t0 + r * kRadixThreads + tid;
    const bool valid = i < n;
    const uint64_t key = valid ? kin[i] : 0ull;
    const int val = valid ? vin[i] : 0;
    const int d = valid ? (int)((key >> shift) & 255) : 256;
#pragma unroll
    for (int ww = 0; ww < kRadixThreads / 32; ++ww) wcnt[ww][tid] = 0;
    __syncthreads();
    const unsigned mask = __match_any_sync(0xffffffffu, d);
    const int rank = __popc(mask & lt);
    if (valid && rank == 0) wcnt[w][d] = __popc(mask);
    __syncthreads();
    int run = 0;
#pragma unroll
    for (int ww = 0; ww < kRadixThreads / 32; ++ww) {
      const int c = wcnt[ww][tid];
      wcnt[ww][tid] = run;
      run += c;
    }
    __syncthreads();
    if (valid) {
      const int pos = base[d] + wcnt[w][d] + rank;
      kout[pos] = key;
      vout[pos] = val;
    }
    __syncthreads();
    base[tid] += run;
    __syncthreads();
  }
}

// ---------------------------------------------------------------- a3
struct Cells {
  int cap = 0;
  int *level = nullptr, *ix = nullptr, *iy = nullptr, *start = nullptr, *count = nullptr,
      *parent = nullptr, *first_child = nullptr, *nchild = nullptr, *leaf = nullptr;
};

int cells_reserve(ddm_ctx_s* ctx, Cells& c, int need, int used, cudaStream_t s) {
  if (need <= c.cap) return DDM_OK;
  int ncap = std::max(need, 2 * c.cap);
  int** fields[9] = {&c.level, &c.ix, &c.iy, &c.start, &c.count, &c.parent, &c.first_child,
                     &c.nchild, &c.leaf};
  for (int f = 0; f < 9; ++f) {
    int* nb = nullptr;
    int rc = talloc(ctx, &nb, ncap, s);
    if (rc) return rc;
    if (*fields[f] && used) DDM_CUDA(ctx, cudaMemcpyAsync(nb, *fields[f], sizeof(int) * used,
                                                          cudaMemcpyDeviceToDevice, s));
    if (*fields[f]) cudaFreeAsync(*fields[f], s);   // stream-ordered after the copy
    *fields[f] = nb;
  }
  c.cap = ncap;
  return DDM_OK;
}

__global__ void split_flags(const uint64_t* __restrict__ keys, const int* __restrict__ cur,
                            const int* __restrict__ c_start, int64_t n, int sh,
                            int* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int c = cur[i];
  int f = 0;
  if (c >= 0) f = (i == c_start[c]) || ((keys[i] >> sh) != (keys[i - 1] >> sh));
  flag[i] = f;
}

__global__ void create_cells(const uint64_t* __restrict__ keys, const int* __restrict__ cur,
                             const int* __restrict__ flag, const int* __restrict__ pos,
                             int64_t n, int sh, int lev, int base, Cells c) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int id = base + pos[i];
  const int par = cur[i];
  const uint64_t pre = keys[i] >> sh;
  c.level[id] = lev;
  c.ix[id] = (int)compact_bits(pre);
  c.iy[id] = (int)compact_bits(pre >> 1);
  c.start[id] = (int)i;
  c.parent[id] = par;
  c.first_child[id] = -1;
  c.nchild[id] = 0;
  if (i == c.start[par]) c.first_child[par] = id;
}

// the root cell (index 0): level 0, the whole sorted range
__global__ void root_cell_init(Cells c, int n, int root_leaf) {
  c.level[0] = 0;
  c.ix[0] = 0;
  c.iy[0] = 0;
  c.start[0] = 0;
  c.count[0] = n;
  c.parent[0] = -1;
  c.first_child[0] = -1;
  c.nchild[0] = 0;
  c.leaf[0] = root_leaf;
}

__global__ void finish_cells(int base, int m, int leaf, int lev, int lmax, Cells c,
                             int* __restrict__ nsplit, int* __restrict__ geom_bad) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= m) return;
  const int id = base + j;
  const int par = c.parent[id];
  const bool last = (j + 1 == m) || (c.parent[id + 1] != par);
  const int end = last ? c.start[par] + c.count[par] : c.start[id + 1];
  const int cnt = end - c.start[id];
  c.count[id] = cnt;
  if (last) c.nchild[par] = id - c.first_child[par] + 1;
  const bool is_leaf = (cnt <= leaf) || (lev >= lmax);
  c.leaf[id] = is_leaf ? 1 : 0;
  if (!is_leaf) atomicAdd(nsplit, 1);
  if (cnt > leaf && lev >= kLBits && lmax >= kLBits) atomicOr(geom_bad, 1);
}

__global__ void update_cur(int* __restrict__ cur, const int* __restrict__ flag,
                           const int* __restrict__ pos, int64_t n, int base,
                           const int* __restrict__ leaf) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  if (cur[i] < 0) return;
  const int child = base + pos[i] + flag[i] - 1;
  cur[i] = leaf[child] ? -1 : child;
}

// ---------------------------------------------------------------- a4
__device__ __forceinline__ bool adj_or_eq(int ax, int ay, int bx, int by) {
  return abs(ax - bx) <= 1 && abs(ay - by) <= 1;
}

// colleagues + V candidates for the cells of one level (lev >= 1)
__global__ void lists_level(int c0, int c1, int lev, const int* __restrict__ parent,
                            const int* __restrict__ ix, const int* __restrict__ iy,
                            const int* __restrict__ first_child, const int* __restrict__ nchild,
                            int* __restrict__ coll, int* __restrict__ vtmp,
                            unsigned char* __restrict__ vcls_tmp, int* __restrict__ vcnt) {
  const int c = c0 + blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= c1) return;
  const int P = parent[c];
  const int cx = ix[c], cy = iy[c];
  int nc = 0, nv = 0;
  for (int k = 0; k < 9; ++k) {
    const int Q = coll[P * 9 + k];
    if (Q < 0) break;
    const int f = first_child[Q], m = nchild[Q];
    for (int q = f; q < f + m; ++q) {
      const int qx = ix[q], qy = iy[q];
      if (adj_or_eq(qx, qy, cx, cy)) {
        coll[c * 9 + nc++] = q;
      } else if (lev >= 2) {
        vtmp[(int64_t)c * 27 + nv] = q;
        vcls_tmp[(int64_t)c * 27 + nv] = (unsigned char)((qy - cy + 3) * 7 + (qx - cx + 3));
        ++nv;
      }
    }
  }
  for (int k = nc; k < 9; ++k) coll[c * 9 + k] = -1;
  vcnt[c] = nv;
}

__global__ void compact_v(int ncells, const int* __restrict__ vtmp,
                          const unsigned char* __restrict__ vcls_tmp,
                          const int* __restrict__ vcnt, const int* __restrict__ voff,
                          int* __restrict__ vidx, unsigned char* __restrict__ vcls) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= ncells) return;
  const int o = voff[c];
  for (int k = 0; k < vcnt[c]; ++k) {
    vidx[o + k] = vtmp[(int64_t)c * 27 + k];
    vcls[o + k] = vcls_tmp[(int64_t)c * 27 + k];
  }
}

__global__ void scatter_leaves(int ncells, const int* __restrict__ leaf,
                               const int* __restrict__ pos, const int* __restrict__ start,
                               int* __restrict__ leaf_by_start) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c < ncells && leaf[c]) leaf_by_start[start[c]] = c;
}

// leaves in element (Morton) order: walk the element-indexed marker array
__global__ void gather_leaves(int64_t n, const int* __restrict__ leaf_by_start,
                              const int* __restrict__ is_start, const int* __restrict__ pos,
                              int* __restrict__ leaves) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n && is_start[i]) leaves[pos[i]] = leaf_by_start[i];
}

__global__ void leaf_start_flags(int64_t n, const int* __restrict__ leaf_by_start,
                                 int* __restrict__ flag) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i < n) flag[i] = leaf_by_start[i] >= 0 ? 1 : 0;
}

__global__ void element_leaf(int nleaves, const int* __restrict__ leaves,
                             const int* __restrict__ start, const int* __restrict__ count,
                             int* __restrict__ el_leaf) {
  const int k = blockIdx.x;
  if (k >= nleaves) return;
  const int c = leaves[k];
  for (int i = threadIdx.x; i < count[c]; i += blockDim.x) el_leaf[start[c] + i] = k;
}

// Enumerate the near field of leaf B (reading R5, W split of SURVEY §8f f3):
//  (1) leaf colleagues of every ancestor of B (incl. B itself) -> U;
//  (2) the subtrees of the non-leaf colleagues of B, walked: a cell touching
//      B is descended (a touching leaf -> U); a non-touching cell D is
//      well separated from B: D -> W (M2P) if count(D) >= w_min, else its
//      whole subtree -> U.  w_min <= 0: (2) puts every subtree in U.
// Returns the number of U ranges; *nw = number of W cells.
__device__ __forceinline__ bool cells_touch(int la, int ixa, int iya, int lb, int ixb, int iyb) {
  if (la > lb) {
    const int t0 = la, t1 = ixa, t2 = iya;
    la = lb; ixa = ixb; iya = iyb;
    lb = t0; ixb = t1; iyb = t2;
  }
  const int sh = lb - la;   // b is the finer cell
  const long long lx = (long long)ixa << sh, hx = (long long)(ixa + 1) << sh;
  const long long ly = (long long)iya << sh, hy = (long long)(iya + 1) << sh;
  return lx <= ixb + 1 && ixb <= hx && ly <= iyb + 1 && iyb <= hy;
}

template <bool kFill>
__device__ int enum_uw(int B, const int* parent, const int* coll, const int* leaf,
                       const int* start, const int* count, const int* level, const int* ix,
                       const int* iy, const int* first_child, const int* nchild, int w_min,
                       int2* out, int* wout, int* nw) {
  int n = 0, m = 0;
  const int lB = level[B], xB = ix[B], yB = iy[B];
  for (int A = B; A >= 0; A = parent[A]) {
    for (int k = 0; k < 9; ++k) {
      const int Q = coll[A * 9 + k];
      if (Q < 0) break;
      if (leaf[Q]) {
        if (kFill) out[n] = make_int2(start[Q], start[Q] + count[Q]);
        ++n;
      } else if (A == B) {
        if (w_min <= 0) {
          if (kFill) out[n] = make_int2(start[Q], start[Q] + count[Q]);
          ++n;
          continue;
        }
        // walk Q's subtree (explicit stack, depth-first)
        int stack[128];
        int sp = 0;
        for (int c = nchild[Q] - 1; c >= 0; --c) stack[sp++] = first_child[Q] + c;
        while (sp > 0) {
          const int D = stack[--sp];
          if (cells_touch(lB, xB, yB, level[D], ix[D], iy[D])) {
            if (leaf[D]) {
              if (kFill) out[n] = make_int2(start[D], start[D] + count[D]);
              ++n;
            } else {
              for (int c = nchild[D] - 1; c >= 0 && sp < 128; --c) stack[sp++] = first_child[D] + c;
            }
          } else if (count[D] >= w_min) {
            if (kFill) wout[m] = D;
            ++m;
          } else {
            if (kFill) out[n] = make_int2(start[D], start[D] + count[D]);
            ++n;
          }
        }
      }
    }
  }
  *nw = m;
  return n;
}

__global__ void u_count(int nleaves, const int* __restrict__ leaves, const int* parent,
                        const int* coll, const int* leaf, const int* start, const int* count,
                        const int* level, const int* ix, const int* iy, const int* first_child,
                        const int* nchild, int w_min, int* __restrict__ ucnt,
                        int* __restrict__ wcnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  int nw = 0;
  ucnt[k] = enum_uw<false>(leaves[k], parent, coll, leaf, start, count, level, ix, iy,
                           first_child, nchild, w_min, nullptr, nullptr, &nw);
  wcnt[k] = nw;
}

__global__ void u_fill(int nleaves, const int* __restrict__ leaves, const int* parent,
                       const int* coll, const int* leaf, const int* start, const int* count,
                       const int* level, const int* ix, const int* iy, const int* first_child,
                       const int* nchild, int w_min, const int* __restrict__ uoff,
                       int2* __restrict__ utmp, int* __restrict__ mcnt, int* __restrict__ nsrc,
                       const int* __restrict__ woff, int* __restrict__ widx) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  int2* r = utmp + uoff[k];
  int* w = widx + woff[k];
  int nw = 0;
  const int n = enum_uw<true>(leaves[k], parent, coll, leaf, start, count, level, ix, iy,
                              first_child, nchild, w_min, r, w, &nw);
  for (int a = 1; a < n; ++a) {  // insertion sort by lo (ranges are disjoint)
    const int2 v = r[a];
    int b = a - 1;
    while (b >= 0 && r[b].x > v.x) { r[b + 1] = r[b]; --b; }
    r[b + 1] = v;
  }
  for (int a = 1; a < nw; ++a) {  // W cells in canonical (index) order
    const int v = w[a];
    int b = a - 1;
    while (b >= 0 && w[b] > v) { w[b + 1] = w[b]; --b; }
    w[b + 1] = v;
  }
  int m = 0, tot = 0;
  for (int a = 0; a < n; ++a) {
    tot += r[a].y - r[a].x;
    if (m > 0 && r[m - 1].y == r[a].x) r[m - 1].y = r[a].y;
    else r[m++] = r[a];
  }
  mcnt[k] = m;
  nsrc[k] = tot;
}

__global__ void u_compact(int nleaves, const int* __restrict__ uoff, const int2* __restrict__ utmp,
                          const int* __restrict__ moff, const int* __restrict__ mcnt,
                          int* __restrict__ lo, int* __restrict__ hi) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  for (int a = 0; a < mcnt[k]; ++a) {
    const int2 v = utmp[uoff[k] + a];
    lo[moff[k] + a] = v.x;
    hi[moff[k] + a] = v.y;
  }
}

// X(B) of leaf B (oracle/tree.py x_lists): the leaf
// colleagues of B's proper ancestors (coarser U-pair leaves) that do not
// touch B, when count(B) >= x_min.  Filled in ascending element start.
__global__ void x_count(int nleaves, const int* __restrict__ leaves, const int* parent,
                        const int* coll, const int* leaf, const int* count, const int* level,
                        const int* ix, const int* iy, int x_min, int* __restrict__ xcnt) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int B = leaves[k];
  int n = 0;
  if (x_min > 0 && count[B] >= x_min) {
    const int lB = level[B], xB = ix[B], yB = iy[B];
    for (int A = parent[B]; A >= 0; A = parent[A])
      for (int q = 0; q < 9; ++q) {
        const int Q = coll[A * 9 + q];
        if (Q < 0) break;
        if (leaf[Q] && !cells_touch(lB, xB, yB, level[Q], ix[Q], iy[Q])) ++n;
      }
  }
  xcnt[k] = n;
}

__global__ void x_fill(int nleaves, const int* __restrict__ leaves, const int* parent,
                       const int* coll, const int* leaf, const int* start, const int* count,
                       const int* level, const int* ix, const int* iy, int x_min,
                       const int* __restrict__ xoff, int* __restrict__ xidx) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int B = leaves[k];
  int* out = xidx + xoff[k];
  const int n = xoff[k + 1] - xoff[k];
  if (n == 0) return;
  const int lB = level[B], xB = ix[B], yB = iy[B];
  int m = 0;
  for (int A = parent[B]; A >= 0; A = parent[A])
    for (int q = 0; q < 9; ++q) {
      const int Q = coll[A * 9 + q];
      if (Q < 0) break;
      if (leaf[Q] && !cells_touch(lB, xB, yB, level[Q], ix[Q], iy[Q])) out[m++] = Q;
    }
  for (int a = 1; a < m; ++a) {   // ascending element start (disjoint leaves)
    const int v = out[a];
    int b = a - 1;
    while (b >= 0 && start[out[b]] > start[v]) { out[b + 1] = out[b]; --b; }
    out[b + 1] = v;
  }
}

__global__ void x_slot_fill(int nleaves, const int* __restrict__ leaves,
                            const int* __restrict__ xoff, int* __restrict__ x_slot) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < nleaves && xoff[k + 1] > xoff[k]) x_slot[leaves[k]] = k;
}

// U(B) minus the element ranges of X(B) (each X leaf lies inside one merged
// U range): kFill = false counts the ranges and the P2P pairs, true writes them
template <bool kFill>
__global__ void ux_ranges(int nleaves, const int* __restrict__ leaves, const int* __restrict__ count,
                          const int* __restrict__ start, const int* __restrict__ u_off,
                          const int* __restrict__ u_lo, const int* __restrict__ u_hi,
                          const int* __restrict__ xoff, const int* __restrict__ xidx,
                          int* __restrict__ cnt, long long* __restrict__ pairs,
                          const int* __restrict__ ux_off, int* __restrict__ ux_lo,
                          int* __restrict__ ux_hi) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int x0 = xoff[k], x1 = xoff[k + 1];
  int n = 0;
  long long src = 0;
  int xi = x0;
  int o = kFill ? ux_off[k] : 0;
  for (int r = u_off[k]; r < u_off[k + 1]; ++r) {
    int cur = u_lo[r];
    const int hi = u_hi[r];
    while (xi < x1 && start[xidx[xi]] < hi) {
      const int a = start[xidx[xi]], b = a + count[xidx[xi]];
      if (a > cur) {
        if (kFill) { ux_lo[o] = cur; ux_hi[o] = a; ++o; }
        ++n;
        src += a - cur;
      }
      cur = b;
      ++xi;
    }
    if (cur < hi) {
      if (kFill) { ux_lo[o] = cur; ux_hi[o] = hi; ++o; }
      ++n;
      src += hi - cur;
    }
  }
  if (!kFill) {
    cnt[k] = n;
    pairs[k] = src * count[leaves[k]];
  }
}

__global__ void item_count(int nleaves, const int* __restrict__ leaves,
                           const int* __restrict__ count, const int* __restrict__ nsrc,
                           int* __restrict__ icnt, long long* __restrict__ pairs) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int nt = count[leaves[k]];
  const int groups = (nt + kTgtGroup - 1) / kTgtGroup;
  const int chunks = max(1, (nsrc[k] + kSrcChunk - 1) / kSrcChunk);
  icnt[k] = groups * chunks;
  pairs[k] = (long long)nt * nsrc[k];
}

// item = (leaf k, first target (sorted index), src_begin, src_end) with the
// source interval in the leaf's concatenated range space [0, nsrc)
__global__ void item_fill(int nleaves, const int* __restrict__ leaves,
                          const int* __restrict__ start, const int* __restrict__ count,
                          const int* __restrict__ nsrc, const int* __restrict__ ioff,
                          int4* __restrict__ items) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const int c = leaves[k];
  const int nt = count[c];
  const int groups = (nt + kTgtGroup - 1) / kTgtGroup;
  const int ns = nsrc[k];
  const int chunks = max(1, (ns + kSrcChunk - 1) / kSrcChunk);
  int o = ioff[k];
  for (int g = 0; g < groups; ++g)
    for (int h = 0; h < chunks; ++h) {
      const int b = (int)((long long)ns * h / chunks);
      const int e = (int)((long long)ns * (h + 1) / chunks);
      items[o++] = make_int4(k, start[c] + g * kTgtGroup, b, e);
    }
}

__global__ void permute_elements(int64_t n, const int* __restrict__ perm,
                                 const double* __restrict__ xc, const double* __restrict__ yc,
                                 const double* __restrict__ a, const double* __restrict__ beta,
                                 double* ex, double* ey, double* ea, double* ec, double* es) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int j = perm[i];
  ex[i] = xc[j];
  ey[i] = yc[j];
  ea[i] = a[j];
  double sb, cb;
  sincos(beta[j], &sb, &cb);
  ec[i] = cb;
  es[i] = sb;
}

__global__ void leaf_cost(int nleaves, const int* __restrict__ leaves,
                          const int* __restrict__ count, const int* __restrict__ nsrc, int p,
                          long long* __restrict__ cost) {
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= nleaves) return;
  const long long nt = count[leaves[k]];
  cost[k] = nt * ((long long)nsrc[k] + p);
}

inline unsigned nblk(int64_t n, int t) { return (unsigned)((n + t - 1) / t); }

}  // namespace

// Host-side split of per-leaf costs into `world` contiguous ranges of near
// equal cost.  split[r] = first leaf of rank r, split[world] = n.
void split_costs(const int64_t* prefix_excl, int64_t total, int nleaves, int world,
                 int* split) {
  split[0] = 0;
  int k = 0;
  for (int r = 1; r < world; ++r) {
    const long double target = (long double)total * r / world;
    while (k < nleaves && (long double)prefix_excl[k] < target) ++k;
    split[r] = std::max(k, split[r - 1]);
  }
  split[world] = nleaves;
}

void free_tree(ddm_tree_s* t) {
  void* ptrs[] = {t->keys_user, t->keys, t->perm, t->ex, t->ey, t->ea, t->ec, t->es,
                  t->el_leaf, t->c_level, t->c_ix, t->c_iy, t->c_start, t->c_count,
                  t->c_parent, t->c_first_child, t->c_nchild, t->c_leaf, t->colleagues,
                  t->v_off, t->v_idx, t->v_cls, t->leaves, t->u_off, t->u_lo, t->u_hi, t->w_off, t->w_idx,
                  t->items, t->item_off, t->p2p_order, t->op_pas, t->op_pasT, t->op_pm2l, t->op_w,
                  t->op_eps, t->op_e2i, t->mpole, t->local, t->src, t->part, t->d_sorted, t->y_sorted, t->y_far,
                  t->up_list,
                  t->krylov, t->pc, t->gm_w, t->gm_tmp, t->gm_part, t->bb_w, t->bb_f,
                  t->pc_chunks, t->pc_off, t->pcl, t->st_elem, t->st_code, t->rbeg, t->srec, t->nc, t->nc_off, t->gm_dev, t->gm_ticket, t->sub_up, t->sub_cells, t->it_roff, t->it_rng, t->gpart, t->lr_rng, t->y_near, t->leaf_info, t->xr_cells, t->xr_off_dev, t->up_own, t->up_strad, t->xsend, t->xrecv, t->ag_send, t->ag_recv, t->ag_lo, t->halo_rng, t->halo_pre, t->dn_own, t->leaf_geo, t->w_geo, t->l2p_runs, t->l2p_order, t->p2p_leaf_order, t->p2m_runs, t->p2m_runs_own, t->x_off, t->x_idx, t->ux_off, t->ux_lo, t->ux_hi, t->lr_rng_x, t->leaf_info_x, t->local_x, t->x_slot};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  if (t->gm_pin) cudaFreeHost(t->gm_pin);
  for (double* p : t->hc_alloc)
    if (p) cudaFree(p);
  if (t->hc_ptrs) cudaFree(t->hc_ptrs);
  for (auto& g : t->graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  if (t->gm_exec) cudaGraphExecDestroy(t->gm_exec);
}

// CUDA events at the stage boundaries of build_tree (ddm_tree_build_times)
struct BuildEvents {
  cudaEvent_t ev[DDM_TB_TOTAL + 1] = {};
  void record(int k, cudaStream_t s) {
    if (!ev[k] && cudaEventCreate(&ev[k]) != cudaSuccess) {
      cudaGetLastError();
      ev[k] = nullptr;
      return;
    }
    cudaEventRecord(ev[k], s);
  }
  void store(double* ms) {
    for (int k = 0; k < DDM_TB_TOTAL; ++k) {
      float v = 0.f;
      if (ev[k] && ev[k + 1] && cudaEventElapsedTime(&v, ev[k], ev[k + 1]) != cudaSuccess) {
        cudaGetLastError();
        v = 0.f;
      }
      ms[k] = v;
    }
  }
  ~BuildEvents() {
    for (auto e : ev)
      if (e) cudaEventDestroy(e);
  }
};

int build_tree(ddm_ctx_s* ctx, const double* xc, const double* yc, const double* a,
               const double* beta, int64_t n, int leaf, int p, double min_side,
               cudaStream_t s, ddm_tree_s* t) {
  if (n < 1 || n > (int64_t)0x7fffffff) return set_error(ctx, DDM_ERR_ARG, "n out of range");
  if (leaf < 1) return set_error(ctx, DDM_ERR_ARG, "leaf_size < 1");
  if (p < 2 || p > kMaxP) return set_error(ctx, DDM_ERR_ARG, "order_p out of [2, 40]");
  int rc;
  t->ctx = ctx;
  t->n = n;
  t->leaf = leaf;
  t->p = p;

  // ---- a1: root square, validation and the largest half-length (one pass,
  // one small read-back)
  BuildEvents bev;
  bev.record(0, s);
  const int mmb = 148;
  double4* part = nullptr;
  double* pamax = nullptr;
  int* dbad = nullptr;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&part, mmb * sizeof(double4), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&pamax, mmb * sizeof(double), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&dbad, sizeof(int), s));
  DDM_CUDA(ctx, cudaMemsetAsync(dbad, 0, sizeof(int), s));
  minmax_partial<<<mmb, 256, 0, s>>>(xc, yc, a, n, part, pamax, dbad);
  DDM_CUDA(ctx, cudaGetLastError());
  std::vector<double4> hpart(mmb);
  std::vector<double> hamax(mmb);
  int hbad = 0;
  DDM_CUDA(ctx, cudaMemcpyAsync(hpart.data(), part, mmb * sizeof(double4),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(hamax.data(), pamax, mmb * sizeof(double),
                                cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaMemcpyAsync(&hbad, dbad, sizeof(int), cudaMemcpyDeviceToHost, s));
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  cudaFreeAsync(part, s);
  cudaFreeAsync(pamax, s);
  cudaFreeAsync(dbad, s);
  if (hbad & 1) return set_error(ctx, DDM_ERR_GEOM, "non-finite element coordinates");
  if (hbad & 2) return set_error(ctx, DDM_ERR_GEOM, "element half-lengths must be finite and > 0");
  double xmn = INFINITY, xmx = -INFINITY, ymn = INFINITY, ymx = -INFINITY;
  t->a_max = 0.0;
  for (int b = 0; b < mmb; ++b) {
    const double4 v = hpart[b];
    xmn = std::min(xmn, v.x); xmx = std::max(xmx, v.y);
    ymn = std::min(ymn, v.z); ymx = std::max(ymx, v.w);
    t->a_max = std::max(t->a_max, hamax[b]);
  }
  double W = std::max(xmx - xmn, ymx - ymn);
  if (W == 0.0) W = 1.0;
  const double scale = 1073741824.0 / W;  // 2^30 / W, one IEEE division
  t->x_min = xmn;
  t->y_min = ymn;
  t->W = W;
  int lmax = kLBits;
  if (min_side > 0.0) lmax = std::max(0, std::min(kLBits, (int)std::floor(std::log2(W / min_side))));

  // ---- a1 keys, a2 sort
  uint64_t* k2 = nullptr;
  int* v2 = nullptr;
  int* vin = nullptr;
  if ((rc = talloc(ctx, &t->keys_user, n, s)) || (rc = talloc(ctx, &t->keys, n, s)) ||
      (rc = talloc(ctx, &t->perm, n, s)))
    return rc;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&k2, n * sizeof(uint64_t), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&v2, n * sizeof(int), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&vin, n * sizeof(int), s));
  morton_kernel<<<nblk(n, 256), 256, 0, s>>>(xc, yc, n, xmn, ymn, scale, t->keys_user, vin);
  DDM_CUDA(ctx, cudaGetLastError());
  bev.record(DDM_TB_SORT, s);
  DDM_CUDA(ctx, cudaMemcpyAsync(t->keys, t->keys_user, n * sizeof(uint64_t),
                                cudaMemcpyDeviceToDevice, s));
  {
    const int nb = (int)nblk(n, kRadixTile);
    int* hist = nullptr;
    int* offs = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&hist, sizeof(int) * 256 * nb, s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&offs, sizeof(int) * 256 * nb, s));
    uint64_t* ka = t->keys;
    int* va = vin;
    uint64_t* kb = k2;
    int* vb = v2;
    for (int pass = 0; pass < 8; ++pass) {  // 60-bit keys: 8 x 8-bit digits
      const int shift = 8 * pass;
      radix_hist<<<nb, 256, 0, s>>>(ka, n, shift, hist, nb);
      DDM_CUDA(ctx, cudaGetLastError());
      if ((rc = exclusive_scan_i32(ctx, hist, offs, 256 * nb, nullptr, s))) return rc;
      radix_scatter<<<nb, kRadixThreads, 0, s>>>(ka, va, kb, vb, n, shift, offs, nb);
      DDM_CUDA(ctx, cudaGetLastError());
      std::swap(ka, kb);
      std::swap(va, vb);
    }
    // 8 passes: result back in t->keys / vin
    DDM_CUDA(ctx, cudaMemcpyAsync(t->perm, va, n * sizeof(int), cudaMemcpyDeviceToDevice, s));
    cudaFreeAsync(hist, s);
    cudaFreeAsync(offs, s);
  }
  cudaFreeAsync(k2, s);
  cudaFreeAsync(v2, s);
  cudaFreeAsync(vin, s);

  // ---- a3 cells, level by level
  bev.record(DDM_TB_CELLS, s);
  Cells C;
  if ((rc = cells_reserve(ctx, C, (int)std::max<int64_t>(64, 4 * (n / leaf + 1) + 8), 0, s)))
    return rc;
  root_cell_init<<<1, 1, 0, s>>>(C, (int)n, (n <= leaf || lmax == 0) ? 1 : 0);
  DDM_CUDA(ctx, cudaGetLastError());
  t->level_off.assign(1, 0);
  t->level_off.push_back(1);
  int ncells = 1;
  {
    int *cur = nullptr, *flag = nullptr, *pos = nullptr, *dsplit = nullptr, *dgeom = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&cur, n * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&flag, n * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&pos, n * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&dsplit, sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&dgeom, sizeof(int), s));
    DDM_CUDA(ctx, cudaMemsetAsync(dgeom, 0, sizeof(int), s));
    const bool root_split = !(n <= leaf || lmax == 0);
    DDM_CUDA(ctx, cudaMemsetAsync(cur, root_split ? 0 : 0xff, n * sizeof(int), s));
    // A level is processed while the previous one split a cell.  Whether it
    // did is read from the next level's scan total (no cell splits <=> no
    // element is flagged, m = 0), so each level costs one host read-back
    // (the scan total) instead of two; the split counter of the last level is
    // read once after the loop, for the depth check.
    int nsplit = root_split ? 1 : 0;
    int lev = 0;
    for (; nsplit > 0 && lev < kLBits; ++lev) {
      const int sh = 2 * (kLBits - lev - 1);
      split_flags<<<nblk(n, 256), 256, 0, s>>>(t->keys, cur, C.start, n, sh, flag);
      DDM_CUDA(ctx, cudaGetLastError());
      int m = 0;
      if ((rc = exclusive_scan_i32(ctx, flag, pos, (int)n, &m, s))) return rc;
      if (m == 0) {   // the previous level split nothing
        nsplit = 0;
        break;
      }
      if ((rc = cells_reserve(ctx, C, ncells + m, ncells, s))) return rc;
      create_cells<<<nblk(n, 256), 256, 0, s>>>(t->keys, cur, flag, pos, n, sh, lev + 1,
                                                ncells, C);
      DDM_CUDA(ctx, cudaGetLastError());
      DDM_CUDA(ctx, cudaMemsetAsync(dsplit, 0, sizeof(int), s));
      finish_cells<<<nblk(m, 256), 256, 0, s>>>(ncells, m, leaf, lev + 1, lmax, C, dsplit,
                                                dgeom);
      DDM_CUDA(ctx, cudaGetLastError());
      update_cur<<<nblk(n, 256), 256, 0, s>>>(cur, flag, pos, n, ncells, C.leaf);
      DDM_CUDA(ctx, cudaGetLastError());
      ncells += m;
      t->level_off.push_back(ncells);
    }
    int hgeom = 0;
    DDM_CUDA(ctx, cudaMemcpyAsync(&hgeom, dgeom, sizeof(int), cudaMemcpyDeviceToHost, s));
    if (nsplit > 0)   // the loop stopped at kLBits levels: did the last one still split?
      DDM_CUDA(ctx, cudaMemcpyAsync(&nsplit, dsplit, sizeof(int), cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    cudaFreeAsync(cur, s);
    cudaFreeAsync(flag, s);
    cudaFreeAsync(pos, s);
    cudaFreeAsync(dsplit, s);
    cudaFreeAsync(dgeom, s);
    if (hgeom || nsplit > 0)
      return set_error(ctx, DDM_ERR_GEOM,
                       "more than leaf_size coincident element centres at the depth cap");
  }
  t->nlevels = (int)t->level_off.size() - 1;
  t->ncells = ncells;
  t->c_level = C.level; t->c_ix = C.ix; t->c_iy = C.iy; t->c_start = C.start;
  t->c_count = C.count; t->c_parent = C.parent; t->c_first_child = C.first_child;
  t->c_nchild = C.nchild; t->c_leaf = C.leaf;

  // ---- a4 colleagues and V lists
  bev.record(DDM_TB_LISTS, s);
  int* vtmp = nullptr;
  unsigned char* vcls_tmp = nullptr;
  int* vcnt = nullptr;
  if ((rc = talloc(ctx, &t->colleagues, (size_t)ncells * 9, s))) return rc;
  if ((rc = talloc(ctx, &t->v_off, ncells + 1, s))) return rc;
  DDM_CUDA(ctx, cudaMallocAsync((void**)&vtmp, (size_t)ncells * 27 * sizeof(int), s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&vcls_tmp, (size_t)ncells * 27, s));
  DDM_CUDA(ctx, cudaMallocAsync((void**)&vcnt, (size_t)(ncells + 1) * sizeof(int), s));
  {
    std::vector<int> rootc(9, -1);
    rootc[0] = 0;
    const int z = 0;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->colleagues, rootc.data(), 9 * sizeof(int),
                                  cudaMemcpyHostToDevice, s));
    DDM_CUDA(ctx, cudaMemcpyAsync(vcnt, &z, sizeof(int), cudaMemcpyHostToDevice, s));
    for (int lev = 1; lev < t->nlevels; ++lev) {
      const int c0 = t->level_off[lev], c1 = t->level_off[lev + 1];
      lists_level<<<nblk(c1 - c0, 128), 128, 0, s>>>(c0, c1, lev, C.parent, C.ix, C.iy,
                                                     C.first_child, C.nchild, t->colleagues,
                                                     vtmp, vcls_tmp, vcnt);
      DDM_CUDA(ctx, cudaGetLastError());
    }
    int nv = 0;
    if ((rc = exclusive_scan_i32(ctx, vcnt, t->v_off, ncells, &nv, s))) return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->v_off + ncells, &nv, sizeof(int), cudaMemcpyHostToDevice, s));
    t->nv = nv;
    if ((rc = talloc(ctx, &t->v_idx, nv, s)) || (rc = talloc(ctx, &t->v_cls, nv, s))) return rc;
    compact_v<<<nblk(ncells, 128), 128, 0, s>>>(ncells, vtmp, vcls_tmp, vcnt, t->v_off,
                                                t->v_idx, t->v_cls);
    DDM_CUDA(ctx, cudaGetLastError());
  }
  cudaFreeAsync(vtmp, s);
  cudaFreeAsync(vcls_tmp, s);
  cudaFreeAsync(vcnt, s);

  // ---- leaves in element order
  {
    int *lbs = nullptr, *flag = nullptr, *pos = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&lbs, n * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&flag, n * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&pos, n * sizeof(int), s));
    DDM_CUDA(ctx, cudaMemsetAsync(lbs, 0xff, n * sizeof(int), s));
    scatter_leaves<<<nblk(ncells, 256), 256, 0, s>>>(ncells, C.leaf, nullptr, C.start, lbs);
    DDM_CUDA(ctx, cudaGetLastError());
    leaf_start_flags<<<nblk(n, 256), 256, 0, s>>>(n, lbs, flag);
    DDM_CUDA(ctx, cudaGetLastError());
    int nl = 0;
    if ((rc = exclusive_scan_i32(ctx, flag, pos, (int)n, &nl, s))) return rc;
    t->nleaves = nl;
    if ((rc = talloc(ctx, &t->leaves, nl, s)) || (rc = talloc(ctx, &t->el_leaf, n, s))) return rc;
    gather_leaves<<<nblk(n, 256), 256, 0, s>>>(n, lbs, flag, pos, t->leaves);
    DDM_CUDA(ctx, cudaGetLastError());
    element_leaf<<<nl, 64, 0, s>>>(nl, t->leaves, C.start, C.count, t->el_leaf);
    DDM_CUDA(ctx, cudaGetLastError());
    cudaFreeAsync(lbs, s);
    cudaFreeAsync(flag, s);
    cudaFreeAsync(pos, s);
  }

  // ---- U lists (merged source ranges), W lists and P2P work items
  if (const char* e = getenv("DDM_W_MIN")) t->w_min = atoi(e);
  {
    const int nl = t->nleaves;
    int *ucnt = nullptr, *uoff = nullptr, *mcnt = nullptr, *moff = nullptr, *nsrc = nullptr;
    int2* utmp = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&ucnt, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&uoff, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&mcnt, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&moff, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&nsrc, nl * sizeof(int), s));
    int* wcnt = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&wcnt, nl * sizeof(int), s));
    u_count<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.parent, t->colleagues, C.leaf,
                                          C.start, C.count, C.level, C.ix, C.iy, C.first_child,
                                          C.nchild, t->w_min, ucnt, wcnt);
    DDM_CUDA(ctx, cudaGetLastError());
    int tot = 0;
    if ((rc = exclusive_scan_i32(ctx, ucnt, uoff, nl, &tot, s))) return rc;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&utmp, (size_t)std::max(tot, 1) * sizeof(int2), s));
    // W lists: offsets per leaf, cells
    int nwt = 0;
    if ((rc = talloc(ctx, &t->w_off, nl + 1, s))) return rc;
    if ((rc = exclusive_scan_i32(ctx, wcnt, t->w_off, nl, &nwt, s))) return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->w_off + nl, &nwt, sizeof(int), cudaMemcpyHostToDevice, s));
    t->nw = nwt;
    if ((rc = talloc(ctx, &t->w_idx, std::max(nwt, 1), s))) return rc;
    u_fill<<<nblk(nl, 64), 64, 0, s>>>(nl, t->leaves, C.parent, t->colleagues, C.leaf, C.start,
                                       C.count, C.level, C.ix, C.iy, C.first_child, C.nchild,
                                       t->w_min, uoff, utmp, mcnt, nsrc, t->w_off, t->w_idx);
    DDM_CUDA(ctx, cudaGetLastError());
    cudaFreeAsync(wcnt, s);
    int nu = 0;
    if ((rc = exclusive_scan_i32(ctx, mcnt, moff, nl, &nu, s))) return rc;
    t->nu = nu;
    if ((rc = talloc(ctx, &t->u_off, nl + 1, s)) || (rc = talloc(ctx, &t->u_lo, nu, s)) ||
        (rc = talloc(ctx, &t->u_hi, nu, s)))
      return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->u_off, moff, nl * sizeof(int), cudaMemcpyDeviceToDevice, s));
    DDM_CUDA(ctx, cudaMemcpyAsync(t->u_off + nl, &nu, sizeof(int), cudaMemcpyHostToDevice, s));
    u_compact<<<nblk(nl, 128), 128, 0, s>>>(nl, uoff, utmp, moff, mcnt, t->u_lo, t->u_hi);
    DDM_CUDA(ctx, cudaGetLastError());

    int* icnt = nullptr;
    long long* pairs = nullptr;
    long long* pairs_scan = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&icnt, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&pairs, nl * sizeof(long long), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&pairs_scan, nl * sizeof(long long), s));
    item_count<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.count, nsrc, icnt, pairs);
    DDM_CUDA(ctx, cudaGetLastError());
    int64_t np = 0;
    if ((rc = exclusive_scan_i64(ctx, (const int64_t*)pairs, (int64_t*)pairs_scan, nl, &np, s)))
      return rc;
    t->near_pairs = np;
    if ((rc = talloc(ctx, &t->item_off, nl + 1, s))) return rc;
    int ni = 0;
    if ((rc = exclusive_scan_i32(ctx, icnt, t->item_off, nl, &ni, s))) return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->item_off + nl, &ni, sizeof(int), cudaMemcpyHostToDevice, s));
    t->nitems = ni;
    if ((rc = talloc(ctx, &t->items, ni, s))) return rc;
    item_fill<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.start, C.count, nsrc, t->item_off,
                                            t->items);
    DDM_CUDA(ctx, cudaGetLastError());

    // per-leaf cost prefix for the multi-GPU partition (kept on host)
    long long* cost = pairs;  // reuse
    leaf_cost<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.count, nsrc, p, cost);
    DDM_CUDA(ctx, cudaGetLastError());
    int64_t ctot = 0;
    if ((rc = exclusive_scan_i64(ctx, (const int64_t*)cost, (int64_t*)pairs_scan, nl, &ctot, s)))
      return rc;
    t->leaf_cost_prefix.assign(nl + 1, 0);
    DDM_CUDA(ctx, cudaMemcpyAsync(t->leaf_cost_prefix.data(), pairs_scan, nl * sizeof(int64_t),
                                  cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    t->leaf_cost_prefix[nl] = ctot;
    cudaFreeAsync(ucnt, s);
    cudaFreeAsync(uoff, s);
    cudaFreeAsync(mcnt, s);
    cudaFreeAsync(moff, s);
    cudaFreeAsync(nsrc, s);
    cudaFreeAsync(utmp, s);
    cudaFreeAsync(icnt, s);
    cudaFreeAsync(pairs, s);
    cudaFreeAsync(pairs_scan, s);
  }

  // ---- X lists and the U ranges without them (elastic series FMM only)
  if (const char* e = getenv("DDM_X_MIN")) t->xl_min = atoi(e);
  if (t->xl_min <= 0) {
    // X lists off (the default): no X entries, U minus X = U -- device copies,
    // no host round trip in the build
    const int nl = t->nleaves;
    t->nx = 0;
    t->nux = t->nu;
    t->near_pairs_x = t->near_pairs;
    if ((rc = talloc(ctx, &t->x_off, nl + 1, s)) || (rc = talloc(ctx, &t->x_idx, 1, s)) ||
        (rc = talloc(ctx, &t->x_slot, (size_t)t->ncells, s)) ||
        (rc = talloc(ctx, &t->ux_off, nl + 1, s)) ||
        (rc = talloc(ctx, &t->ux_lo, std::max<int64_t>(t->nu, 1), s)) ||
        (rc = talloc(ctx, &t->ux_hi, std::max<int64_t>(t->nu, 1), s)))
      return rc;
    DDM_CUDA(ctx, cudaMemsetAsync(t->x_off, 0, (size_t)(nl + 1) * sizeof(int), s));
    DDM_CUDA(ctx, cudaMemsetAsync(t->x_slot, 0xFF, (size_t)t->ncells * sizeof(int), s));
    DDM_CUDA(ctx, cudaMemcpyAsync(t->ux_off, t->u_off, (size_t)(nl + 1) * sizeof(int),
                                  cudaMemcpyDeviceToDevice, s));
    if (t->nu > 0) {
      DDM_CUDA(ctx, cudaMemcpyAsync(t->ux_lo, t->u_lo, (size_t)t->nu * sizeof(int),
                                    cudaMemcpyDeviceToDevice, s));
      DDM_CUDA(ctx, cudaMemcpyAsync(t->ux_hi, t->u_hi, (size_t)t->nu * sizeof(int),
                                    cudaMemcpyDeviceToDevice, s));
    }
  } else {
    const int nl = t->nleaves;
    int *xcnt = nullptr, *uxcnt = nullptr;
    long long *pairs = nullptr, *pairs_scan = nullptr;
    DDM_CUDA(ctx, cudaMallocAsync((void**)&xcnt, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&uxcnt, nl * sizeof(int), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&pairs, nl * sizeof(long long), s));
    DDM_CUDA(ctx, cudaMallocAsync((void**)&pairs_scan, nl * sizeof(long long), s));
    x_count<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.parent, t->colleagues, C.leaf, C.count,
                                          C.level, C.ix, C.iy, t->xl_min, xcnt);
    DDM_CUDA(ctx, cudaGetLastError());
    int nxt = 0;
    if ((rc = talloc(ctx, &t->x_off, nl + 1, s))) return rc;
    if ((rc = exclusive_scan_i32(ctx, xcnt, t->x_off, nl, &nxt, s))) return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->x_off + nl, &nxt, sizeof(int), cudaMemcpyHostToDevice, s));
    t->nx = nxt;
    if ((rc = talloc(ctx, &t->x_idx, std::max(nxt, 1), s))) return rc;
    x_fill<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.parent, t->colleagues, C.leaf, C.start,
                                         C.count, C.level, C.ix, C.iy, t->xl_min, t->x_off,
                                         t->x_idx);
    DDM_CUDA(ctx, cudaGetLastError());
    if ((rc = talloc(ctx, &t->x_slot, (size_t)t->ncells, s))) return rc;
    DDM_CUDA(ctx, cudaMemsetAsync(t->x_slot, 0xFF, (size_t)t->ncells * sizeof(int), s));
    x_slot_fill<<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, t->x_off, t->x_slot);
    DDM_CUDA(ctx, cudaGetLastError());
    ux_ranges<false><<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.count, C.start, t->u_off,
                                                   t->u_lo, t->u_hi, t->x_off, t->x_idx, uxcnt,
                                                   pairs, nullptr, nullptr, nullptr);
    DDM_CUDA(ctx, cudaGetLastError());
    int nux = 0;
    if ((rc = talloc(ctx, &t->ux_off, nl + 1, s))) return rc;
    if ((rc = exclusive_scan_i32(ctx, uxcnt, t->ux_off, nl, &nux, s))) return rc;
    DDM_CUDA(ctx, cudaMemcpyAsync(t->ux_off + nl, &nux, sizeof(int), cudaMemcpyHostToDevice, s));
    t->nux = nux;
    if ((rc = talloc(ctx, &t->ux_lo, std::max(nux, 1), s)) ||
        (rc = talloc(ctx, &t->ux_hi, std::max(nux, 1), s)))
      return rc;
    ux_ranges<true><<<nblk(nl, 128), 128, 0, s>>>(nl, t->leaves, C.count, C.start, t->u_off,
                                                  t->u_lo, t->u_hi, t->x_off, t->x_idx, nullptr,
                                                  nullptr, t->ux_off, t->ux_lo, t->ux_hi);
    DDM_CUDA(ctx, cudaGetLastError());
    int64_t npx = 0;
    if ((rc = exclusive_scan_i64(ctx, (const int64_t*)pairs, (int64_t*)pairs_scan, nl, &npx, s)))
      return rc;
    t->near_pairs_x = npx;
    cudaFreeAsync(xcnt, s);
    cudaFreeAsync(uxcnt, s);
    cudaFreeAsync(pairs, s);
    cudaFreeAsync(pairs_scan, s);
  }

  // ---- element data in Morton order
  bev.record(DDM_TB_SCHED, s);
  if ((rc = talloc(ctx, &t->ex, n, s)) || (rc = talloc(ctx, &t->ey, n, s)) ||
      (rc = talloc(ctx, &t->ea, n, s)) || (rc = talloc(ctx, &t->ec, n, s)) ||
      (rc = talloc(ctx, &t->es, n, s)))
    return rc;
  permute_elements<<<nblk(n, 256), 256, 0, s>>>(n, t->perm, xc, yc, a, beta, t->ex, t->ey,
                                                t->ea, t->ec, t->es);
  DDM_CUDA(ctx, cudaGetLastError());

  // ---- upward-pass schedule: non-leaf cells of level >= 2, deepest level
  // first (every parent after all of its children), one range per level
  {
    std::vector<int> hleaf(ncells);
    DDM_CUDA(ctx, cudaMemcpyAsync(hleaf.data(), C.leaf, ncells * sizeof(int),
                                  cudaMemcpyDeviceToHost, s));
    DDM_CUDA(ctx, cudaStreamSynchronize(s));
    std::vector<int> up;
    t->up_level_off.assign(2 * (t->nlevels + 1), 0);
    for (int lev = t->nlevels - 1; lev >= 2; --lev) {
      t->up_level_off[2 * lev] = (int)up.size();
      for (int c = t->level_off[lev]; c < t->level_off[lev + 1]; ++c)
        if (!hleaf[c]) up.push_back(c);
      t->up_level_off[2 * lev + 1] = (int)up.size();
    }
    t->n_up = (int)up.size();
    t->h_up = up;
    if ((rc = talloc(ctx, &t->up_list, up.size(), s))) return rc;
    if (!up.empty())
      DDM_CUDA(ctx, cudaMemcpyAsync(t->up_list, up.data(), up.size() * sizeof(int),
                                    cudaMemcpyHostToDevice, s));

    // subtree schedule (expansions.cu subtree passes): split level Ls = the
    // first level >= 3 with >= 128 cells, if at least two levels lie below it
    int Ls = -1;
    for (int lev = 3; lev < t->nlevels; ++lev)
      if (t->level_off[lev + 1] - t->level_off[lev] >= 128) {
        Ls = lev;
        break;
      }
    t->sub_n = 0;
    std::vector<int2> sup, scell;
    if (Ls > 0 && t->nlevels - 1 - Ls >= 2) {
      std::vector<int> hpar(ncells);
      DDM_CUDA(ctx, cudaMemcpyAsync(hpar.data(), C.parent, ncells * sizeof(int),
                                    cudaMemcpyDeviceToHost, s));
      DDM_CUDA(ctx, cudaStreamSynchronize(s));
      const int nroot = t->level_off[Ls + 1] - t->level_off[Ls];
      const int nsl = t->nlevels - Ls;
      // root of every cell at level >= Ls (parents precede children by level)
      std::vector<int> root(ncells, -1);
      for (int c = t->level_off[Ls]; c < t->level_off[Ls + 1]; ++c) root[c] = c - t->level_off[Ls];
      for (int lev = Ls + 1; lev < t->nlevels; ++lev)
        for (int c = t->level_off[lev]; c < t->level_off[lev + 1]; ++c) root[c] = root[hpar[c]];
      sup.assign((size_t)nroot * nsl, make_int2(0, 0));
      scell.assign((size_t)nroot * nsl, make_int2(0, 0));
      for (int lev = Ls; lev < t->nlevels; ++lev) {
        const int L = lev - Ls;
        for (int c = t->level_off[lev]; c < t->level_off[lev + 1]; ++c) {
          int2& r = scell[(size_t)root[c] * nsl + L];
          if (r.y == r.x) r = make_int2(c, c + 1); else r.y = c + 1;   // contiguous (Morton)
        }
        for (int k = t->up_level_off[2 * lev]; k < t->up_level_off[2 * lev + 1]; ++k) {
          int2& r = sup[(size_t)root[up[k]] * nsl + L];
          if (r.y == r.x) r = make_int2(k, k + 1); else r.y = k + 1;
        }
      }
      // the ranges must be exactly the subtree's entries (Morton contiguity)
      std::vector<int> cnt_c((size_t)nroot * nsl, 0), cnt_u((size_t)nroot * nsl, 0);
      for (int lev = Ls; lev < t->nlevels; ++lev) {
        for (int c = t->level_off[lev]; c < t->level_off[lev + 1]; ++c)
          ++cnt_c[(size_t)root[c] * nsl + (lev - Ls)];
        for (int k = t->up_level_off[2 * lev]; k < t->up_level_off[2 * lev + 1]; ++k)
          ++cnt_u[(size_t)root[up[k]] * nsl + (lev - Ls)];
      }
      bool ok = true;
      for (size_t i = 0; i < cnt_c.size(); ++i)
        ok = ok && cnt_c[i] == scell[i].y - scell[i].x && cnt_u[i] == sup[i].y - sup[i].x;
      if (!ok) Ls = -1;
    }
    if (Ls > 0 && t->nlevels - 1 - Ls >= 2) {
      const int nroot = t->level_off[Ls + 1] - t->level_off[Ls];
      const int nsl = t->nlevels - Ls;
      if ((rc = talloc(ctx, &t->sub_up, sup.size(), s)) || (rc = talloc(ctx, &t->sub_cells, scell.size(), s)))
        return rc;
      DDM_CUDA(ctx, cudaMemcpyAsync(t->sub_up, sup.data(), sup.size() * sizeof(int2),
                                    cudaMemcpyHostToDevice, s));
      DDM_CUDA(ctx, cudaMemcpyAsync(t->sub_cells, scell.data(), scell.size() * sizeof(int2),
                                    cudaMemcpyHostToDevice, s));
      DDM_CUDA(ctx, cudaStreamSynchronize(s));
      t->sub_Ls = Ls;
      t->sub_n = nroot;
      t->sub_nsl = nsl;
    }
  }
  bev.record(DDM_TB_TOTAL, s);
  DDM_CUDA(ctx, cudaStreamSynchronize(s));
  bev.store(t->build_ms);
  return DDM_OK;
}

}  // namespace ddm
