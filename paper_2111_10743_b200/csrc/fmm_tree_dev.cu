// The reference octree (fmm.py:539-647) built on the device, bit-exact with
// the host build in fmm_tree.cpp (and so with `_build_tree`): Morton keys,
// stable radix sort, then a level-synchronous box discovery over the sorted
// keys and the reference's DFS-LIFO numbering computed without a DFS:
//
//   * level L's boxes are the runs of equal 3L-bit key prefix among points
//     whose level-(L-1) box is not a leaf (sorted order keeps each parent's
//     children contiguous and in ascending octant order);
//   * subtree sizes bottom-up, then the preorder position of every box in a
//     DFS that visits children in DESCENDING octant order (the LIFO stack
//     pops the highest octant first): pos(c) = pos(p) + 1 + sizes of the
//     higher-octant siblings;
//   * the reference pops boxes in that preorder and numbers the children of
//     each popped non-leaf consecutively, so
//       id(c) = 1 + (children of non-leaves popped before p) + octant rank,
//     an exclusive scan of child counts in preorder.
#include <cub/cub.cuh>

#include <chrono>

#include <string>
#include <type_traits>
#include <vector>

#include "fmm_plan.h"
#include "lb_common.cuh"

namespace lb {

// fmm.py:569-576 on the device; explicit _rn intrinsics keep the arithmetic
// identical to numpy's (no contraction).  The one definition (round 1 kept it
// in fmm_plan.cu behind a declaration here).
__global__ void morton_keys_kernel(const double* __restrict__ spos, int64_t ns,
                                   const double* __restrict__ tpos, int64_t nt, double c0, double c1,
                                   double c2, double half, uint64_t* __restrict__ keys,
                                   int64_t* __restrict__ idx) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns + nt) return;
  const double* p = i < ns ? spos + 3 * i : tpos + 3 * (i - ns);
  const double cc[3] = {c0, c1, c2};
  const double two_h = __dmul_rn(2.0, half);
  uint64_t code = 0;
#pragma unroll
  for (int a = 0; a < 3; ++a) {
    const double origin = __dsub_rn(cc[a], half);
    const double q = __ddiv_rn(__dsub_rn(p[a], origin), two_h);
    int64_t cell = (int64_t)__dmul_rn(q, (double)(1 << kMaxDepth));
    cell = cell < 0 ? 0 : (cell > (1 << kMaxDepth) - 1 ? (1 << kMaxDepth) - 1 : cell);
    for (int b = 0; b < kMaxDepth; ++b) code |= (uint64_t)((cell >> b) & 1) << (3 * b + a);
  }
  keys[i] = code;
  idx[i] = i;
}

namespace {

constexpr int kT = 256;

inline unsigned blocks(int64_t n) { return (unsigned)std::max<int64_t>(1, ceil_div(n, kT)); }

__device__ __forceinline__ uint64_t prefix(uint64_t code, int lev) { return code >> (3 * (kMaxDepth - lev)); }

// start / end of every level-L box among the points still inside non-leaf boxes
__global__ void level_flags_kernel(const uint64_t* __restrict__ codes, const uint8_t* __restrict__ alive,
                                   int64_t m, int lev, int32_t* __restrict__ start) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m) return;
  int32_t s = 0;
  if (alive[i]) s = (i == 0 || !alive[i - 1] || prefix(codes[i], lev) != prefix(codes[i - 1], lev)) ? 1 : 0;
  start[i] = s;
}

// per point of a new box: its range, parent, key prefix; incl = inclusive scan of start
__global__ void level_boxes_kernel(const uint64_t* __restrict__ codes, const uint8_t* __restrict__ alive,
                                   const int32_t* __restrict__ start, const int32_t* __restrict__ incl,
                                   const int32_t* __restrict__ pbox, int64_t m, int lev, int64_t g0,
                                   int64_t* __restrict__ lo, int64_t* __restrict__ hi,
                                   int32_t* __restrict__ parent, int64_t* __restrict__ ijk,
                                   int32_t* __restrict__ level) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || !alive[i]) return;
  const int64_t g = g0 + incl[i] - 1;
  if (start[i]) {
    lo[g] = i;
    parent[g] = pbox[i];
    level[g] = lev;
    const uint64_t key = prefix(codes[i], lev);
#pragma unroll
    for (int a = 0; a < 3; ++a) {
      int64_t c = 0;
      for (int b = 0; b < lev; ++b) c |= (int64_t)((key >> (3 * b + a)) & 1) << b;
      ijk[3 * g + a] = c;
    }
  }
  const bool end = i == m - 1 || !alive[i + 1] || prefix(codes[i], lev) != prefix(codes[i + 1], lev);
  if (end) hi[g] = i + 1;
}

__global__ void level_leaf_kernel(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi, int64_t g0,
                                  int64_t n, int lev, int ncrit, uint8_t* __restrict__ leaf,
                                  int* __restrict__ overflow) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t g = g0 + j, cnt = hi[g] - lo[g];
  const bool is_leaf = cnt <= ncrit || lev == kMaxDepth;  // fmm.py:600
  leaf[g] = is_leaf ? 1 : 0;
  if (lev == kMaxDepth && cnt > 64 * (int64_t)ncrit) atomicExch(overflow, 1);  // fmm.py:605-609
}

__global__ void level_alive_kernel(const int32_t* __restrict__ incl, const uint8_t* __restrict__ leaf,
                                   int64_t m, int64_t g0, uint8_t* __restrict__ alive,
                                   int32_t* __restrict__ pbox) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= m || !alive[i]) return;
  const int64_t g = g0 + incl[i] - 1;
  pbox[i] = (int32_t)g;
  alive[i] = leaf[g] ? 0 : 1;
}

// first child and child count of every parent (children are contiguous)
__global__ void children_kernel(const int32_t* __restrict__ parent, int64_t g0, int64_t n,
                                int32_t* __restrict__ first, int32_t* __restrict__ nchild) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t g = g0 + j;
  const int32_t p = parent[g];
  if (j == 0 || parent[g - 1] != p) {
    first[p] = (int32_t)g;
    int k = 1;
    while (j + k < n && parent[g + k] == p) ++k;
    nchild[p] = k;
  }
}

__global__ void subtree_kernel(const int32_t* __restrict__ first, const int32_t* __restrict__ nchild,
                               int64_t g0, int64_t n, int32_t* __restrict__ size) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t g = g0 + j;
  int32_t s = 1;
  for (int k = 0; k < nchild[g]; ++k) s += size[first[g] + k];
  size[g] = s;
}

__global__ void preorder_kernel(const int32_t* __restrict__ first, const int32_t* __restrict__ nchild,
                                const int32_t* __restrict__ size, int64_t g0, int64_t n,
                                int32_t* __restrict__ pos) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t g = g0 + j;
  int32_t at = pos[g] + 1;  // highest octant first
  for (int k = nchild[g] - 1; k >= 0; --k) {
    pos[first[g] + k] = at;
    at += size[first[g] + k];
  }
}

__global__ void scatter_by_pos_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ nchild,
                                      int64_t n, int32_t* __restrict__ nc_at_pos) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g < n) nc_at_pos[pos[g]] = nchild[g];
}

__global__ void ids_kernel(const int32_t* __restrict__ pos, const int32_t* __restrict__ first,
                           const int32_t* __restrict__ nchild, const int32_t* __restrict__ base_at_pos,
                           int64_t n, int32_t* __restrict__ id) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  if (g == 0) id[0] = 0;
  const int32_t b = 1 + base_at_pos[pos[g]];
  for (int k = 0; k < nchild[g]; ++k) id[first[g] + k] = b + k;
}

// per-box outputs in reference id order
__global__ void by_id_kernel(const int32_t* __restrict__ id, const int32_t* __restrict__ level_g,
                             const int64_t* __restrict__ ijk_g, const int32_t* __restrict__ parent_g,
                             const uint8_t* __restrict__ leaf_g, const int64_t* __restrict__ lo_g,
                             const int64_t* __restrict__ hi_g, const int32_t* __restrict__ nchild_g,
                             const int64_t* __restrict__ ps, const int64_t* __restrict__ pt, int64_t n,
                             int32_t* __restrict__ level, int64_t* __restrict__ ijk, int64_t* __restrict__ parent,
                             uint8_t* __restrict__ leaf, int64_t* __restrict__ lo, int64_t* __restrict__ hi,
                             int64_t* __restrict__ nchild, int64_t* __restrict__ srng, int64_t* __restrict__ trng) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  const int64_t b = id[g];
  level[b] = level_g[g];
  for (int a = 0; a < 3; ++a) ijk[3 * b + a] = ijk_g[3 * g + a];
  parent[b] = g == 0 ? -1 : id[parent_g[g]];
  leaf[b] = leaf_g[g];
  lo[b] = lo_g[g];
  hi[b] = hi_g[g];
  nchild[b] = nchild_g[g];
  srng[2 * b] = ps[lo_g[g]];
  srng[2 * b + 1] = ps[hi_g[g]];
  trng[2 * b] = pt[lo_g[g]];
  trng[2 * b + 1] = pt[hi_g[g]];
}

__global__ void children_idx_kernel(const int32_t* __restrict__ id, const int32_t* __restrict__ first,
                                    const int32_t* __restrict__ nchild, const int64_t* __restrict__ off_by_id,
                                    int64_t n, int64_t* __restrict__ idx) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n || nchild[g] == 0) return;
  const int64_t o = off_by_id[id[g]];
  for (int k = 0; k < nchild[g]; ++k) idx[o + k] = id[first[g] + k];
}

__global__ void src_flags_kernel(const int64_t* __restrict__ order, int64_t m, int64_t ns,
                                 int64_t* __restrict__ is_src, int64_t* __restrict__ is_tgt) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  const bool s = order[p] < ns;
  is_src[p] = s ? 1 : 0;
  is_tgt[p] = s ? 0 : 1;
}

__global__ void split_kernel(const int64_t* __restrict__ order, const int64_t* __restrict__ ps,
                             const int64_t* __restrict__ pt, int64_t m, int64_t ns,
                             int64_t* __restrict__ src_sorted, int64_t* __restrict__ tgt_sorted) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= m) return;
  const int64_t o = order[p];
  if (o < ns) src_sorted[ps[p]] = o;
  else tgt_sorted[pt[p]] = o - ns;
}


// ---- interaction lists (fmm.py:662-715) in the level-major index space g;
// every list in the reference's order, written as reference box ids

struct GTree {
  const int32_t* lev;
  const int64_t* ijk;
  const int32_t* par;
  const uint8_t* leaf;
  const int32_t* first;
  const int32_t* nchild;
  const int64_t* nsrc;
  const int64_t* ntgt;
  const int32_t* id;
  int32_t* cols;   // (nbox, K) colleagues, g indices
  int32_t* ncol;
  int K, buffer;
};

__device__ __forceinline__ int64_t cheb(const GTree& T, int64_t a, int64_t b) {
  const int64_t dx = llabs(T.ijk[3 * a] - T.ijk[3 * b]), dy = llabs(T.ijk[3 * a + 1] - T.ijk[3 * b + 1]),
                dz = llabs(T.ijk[3 * a + 2] - T.ijk[3 * b + 2]);
  return max(dx, max(dy, dz));
}

// fmm.py:650-659
__device__ __forceinline__ bool near_g(const GTree& T, int64_t a, int64_t b) {
  const int la = T.lev[a], lb = T.lev[b];
  const int lf = max(la, lb);
  const int64_t sa = (int64_t)1 << (lf - la), sb = (int64_t)1 << (lf - lb);
  const int64_t m = min(sa, sb) * T.buffer;
  for (int k = 0; k < 3; ++k) {
    const int64_t alo = T.ijk[3 * a + k] * sa, blo = T.ijk[3 * b + k] * sb;
    const int64_t gap = max(blo - (alo + sa), alo - (blo + sb));
    if (!(gap < m)) return false;
  }
  return true;
}

__global__ void box_counts_kernel(const int64_t* __restrict__ lo, const int64_t* __restrict__ hi,
                                  const int64_t* __restrict__ ps, const int64_t* __restrict__ pt, int64_t n,
                                  int64_t* __restrict__ nsrc, int64_t* __restrict__ ntgt) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  nsrc[g] = ps[hi[g]] - ps[lo[g]];
  ntgt[g] = pt[hi[g]] - pt[lo[g]];
}

// colleagues of level-L boxes and their V-list lengths (fmm.py:669-679)
template <bool FILL>
__global__ void colleagues_kernel(GTree T, int64_t g0, int64_t n, int64_t* __restrict__ vcnt_id,
                                  const int64_t* __restrict__ voff_id, int64_t* __restrict__ vidx) {
  const int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  const int64_t b = g0 + j, p = T.par[b];
  int nc = 0;
  int64_t cv = 0, at = FILL ? voff_id[T.id[b]] : 0;
  for (int q = 0; q < T.ncol[p]; ++q) {
    const int64_t pc = T.cols[p * T.K + q];
    for (int k = 0; k < T.nchild[pc]; ++k) {
      const int64_t c = T.first[pc] + k;
      if (cheb(T, c, b) <= T.buffer) {
        if (!FILL) T.cols[b * T.K + nc] = (int32_t)c;
        ++nc;
      } else if (T.nsrc[c] > 0) {
        if (FILL) vidx[at++] = T.id[c];
        ++cv;
      }
    }
  }
  if (!FILL) {
    T.ncol[b] = nc;
    vcnt_id[T.id[b]] = cv;
  }
}

__global__ void colleague_rows_kernel(GTree T, int64_t n, int64_t* __restrict__ cnt_id,
                                      const int64_t* __restrict__ off_id, int64_t* __restrict__ idx) {
  const int64_t g = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (g >= n) return;
  if (!off_id) {
    cnt_id[T.id[g]] = T.ncol[g];
    return;
  }
  const int64_t o = off_id[T.id[g]];
  for (int q = 0; q < T.ncol[g]; ++q) idx[o + q] = T.id[T.cols[g * T.K + q]];
}

constexpr int kStack = 384;

// U, W and X of the non-empty leaves (fmm.py:684-714); the count pass and
// the fill pass run the same walk
template <bool FILL>
__global__ void uwx_kernel(GTree T, int64_t n, int64_t* __restrict__ ucnt, int64_t* __restrict__ wcnt,
                           int64_t* __restrict__ xcnt, const int64_t* __restrict__ uoff,
                           const int64_t* __restrict__ woff, int64_t* __restrict__ xcur,
                           int64_t* __restrict__ uidx, int64_t* __restrict__ widx, int64_t* __restrict__ xidx,
                           int* __restrict__ overflow) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b >= n || !T.leaf[b]) return;
  const bool has_src = T.nsrc[b] > 0;
  if (!has_src && T.ntgt[b] == 0) return;
  const int64_t bid = T.id[b];
  int64_t nu = 0, nw = 0;
  int64_t* u = FILL ? uidx + uoff[bid] : nullptr;
  int64_t* w = FILL ? widx + woff[bid] : nullptr;
  // colleagues of an ancestor are boxes of its level: no repeats, so the
  // reference's `seen` set never drops one
  for (int64_t a = b; a != -1; a = T.par[a])
    for (int q = 0; q < T.ncol[a]; ++q) {
      const int64_t c = T.cols[a * T.K + q];
      if (T.leaf[c] && c != b && near_g(T, b, c)) {
        if (FILL) u[nu] = T.id[c];
        ++nu;
      }
    }
  if (FILL) u[nu] = bid;
  ++nu;
  int32_t stack[kStack];
  int sp = 0;
  for (int q = 0; q < T.ncol[b]; ++q) {
    const int32_t c = T.cols[b * T.K + q];
    if (!T.leaf[c]) stack[sp++] = c;
  }
  while (sp > 0) {
    const int64_t c = stack[--sp];
    for (int k = 0; k < T.nchild[c]; ++k) {
      const int64_t kk = T.first[c] + k;
      if (near_g(T, b, kk)) {
        if (T.leaf[kk]) {
          if (FILL) u[nu] = T.id[kk];
          ++nu;
        } else if (sp < kStack) {
          stack[sp++] = (int32_t)kk;
        } else {
          atomicExch(overflow, 1);
        }
      } else {
        if (T.nsrc[kk] > 0) {
          if (FILL) w[nw] = T.id[kk];
          ++nw;
        }
        if (has_src) {
          if (FILL) xidx[atomicAdd((unsigned long long*)&xcur[T.id[kk]], 1ull)] = bid;
          else atomicAdd((unsigned long long*)&xcnt[T.id[kk]], 1ull);
        }
      }
    }
  }
  if (!FILL) {
    ucnt[bid] = nu;
    wcnt[bid] = nw;
  }
}

// X[k] in ascending leaf id, the reference's loop order
__global__ void sort_rows_kernel(const int64_t* __restrict__ off, int64_t n, int64_t* __restrict__ idx) {
  const int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (r >= n) return;
  for (int64_t i = off[r] + 1; i < off[r + 1]; ++i) {
    const int64_t v = idx[i];
    int64_t j = i - 1;
    while (j >= off[r] && idx[j] > v) {
      idx[j + 1] = idx[j];
      --j;
    }
    idx[j + 1] = v;
  }
}

// device scratch owned by one build; frees on scope exit
struct TreeScratch {
  std::vector<void*> ptrs;
  cudaError_t err = cudaSuccess;
  template <class T>
  T* get(int64_t n) {
    void* p = nullptr;
    if (err == cudaSuccess) err = cudaMalloc(&p, std::max<size_t>((size_t)n * sizeof(T), 16));
    if (err == cudaSuccess) ptrs.push_back(p);
    return (T*)p;
  }
  template <class T>
  T* release(T* p) {  // hand ownership to the caller
    ptrs.erase(std::remove(ptrs.begin(), ptrs.end(), (void*)p), ptrs.end());
    return p;
  }
  ~TreeScratch() {
    for (void* p : ptrs) cudaFree(p);
  }
};

template <class T>
cudaError_t scan_excl(TreeScratch& S, const T* in, T* out, int64_t n) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::ExclusiveSum(nullptr, bytes, in, out, n);
  void* tmp = S.get<uint8_t>((int64_t)bytes);
  if (e == cudaSuccess) e = S.err;
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(tmp, bytes, in, out, n);
  return e;
}

template <class T>
cudaError_t scan_incl(TreeScratch& S, const T* in, T* out, int64_t n) {
  size_t bytes = 0;
  cudaError_t e = cub::DeviceScan::InclusiveSum(nullptr, bytes, in, out, n);
  void* tmp = S.get<uint8_t>((int64_t)bytes);
  if (e == cudaSuccess) e = S.err;
  if (e == cudaSuccess) e = cub::DeviceScan::InclusiveSum(tmp, bytes, in, out, n);
  return e;
}

template <class T>
cudaError_t d2h(std::vector<T>& dst, const T* src, int64_t n) {
  dst.resize(n);
  return n ? cudaMemcpy(dst.data(), src, (size_t)n * sizeof(T), cudaMemcpyDeviceToHost) : cudaSuccess;
}

}  // namespace

#define TD_TRY(expr)                                                                          \
  do {                                                                                        \
    cudaError_t _e = (expr);                                                                  \
    if (_e == cudaSuccess) _e = S.err;                                                        \
    if (_e == cudaSuccess) _e = cudaGetLastError();                                           \
    if (_e != cudaSuccess) return fail(LB_ERR_CUDA, std::string("fmm device tree: ") + #expr + \
                                                        ": " + cudaGetErrorString(_e));       \
  } while (0)

int tree_build_device(FmmTree& t, const double* spos, const double* tpos, int buffer, double* lists_ms,
                      TreeDev* keep) {
  const int64_t m = t.ns + t.nt;
  if (m >= ((int64_t)1 << 31)) return fail(LB_ERR_SHAPE, "fmm device tree: more than 2^31 points");
  TreeScratch S;
  tree_bounds(spos, t.ns, tpos, t.nt, t.center, &t.half);
  // keys + stable LSD radix sort on the 60 key bits (fmm.py:569-577)
  double* ds = S.get<double>(3 * t.ns);
  double* dt = S.get<double>(3 * t.nt);
  uint64_t* k0 = S.get<uint64_t>(m);
  uint64_t* codes = S.get<uint64_t>(m);
  int64_t* v0 = S.get<int64_t>(m);
  int64_t* order = S.get<int64_t>(m);
  TD_TRY(S.err);
  if (t.ns) TD_TRY(cudaMemcpy(ds, spos, sizeof(double) * 3 * t.ns, cudaMemcpyHostToDevice));
  if (t.nt) TD_TRY(cudaMemcpy(dt, tpos, sizeof(double) * 3 * t.nt, cudaMemcpyHostToDevice));
  morton_keys_kernel<<<blocks(m), kT>>>(ds, t.ns, dt, t.nt, t.center[0], t.center[1], t.center[2], t.half, k0, v0);
  TD_TRY(cudaGetLastError());
  {
    size_t bytes = 0;
    TD_TRY(cub::DeviceRadixSort::SortPairs(nullptr, bytes, k0, codes, v0, order, m, 0, 3 * kMaxDepth));
    void* tmp = S.get<uint8_t>((int64_t)bytes);
    TD_TRY(cub::DeviceRadixSort::SortPairs(tmp, bytes, k0, codes, v0, order, m, 0, 3 * kMaxDepth));
  }
  // level-synchronous boxes, level-major index g (capacity: at most m boxes
  // per level below the root, and at most 2m - 1 in total)
  // per-box arrays grow with the levels (typical trees hold ~m/40 boxes;
  // pathological clustering can reach ~20 m)
  int64_t cap = std::max<int64_t>(4096, m / 8);
  int64_t* lo_g = S.get<int64_t>(cap);
  int64_t* hi_g = S.get<int64_t>(cap);
  int32_t* par_g = S.get<int32_t>(cap);
  int64_t* ijk_g = S.get<int64_t>(3 * cap);
  int32_t* lev_g = S.get<int32_t>(cap);
  uint8_t* leaf_g = S.get<uint8_t>(cap);
  auto grow = [&](int64_t need, int64_t used) -> cudaError_t {
    const int64_t nc = std::max(need, 2 * cap);
    auto move = [&](auto*& p, int64_t per) {
      using T = std::remove_reference_t<decltype(*p)>;
      T* q = S.get<T>(nc * per);
      if (S.err == cudaSuccess && used)
        S.err = cudaMemcpy(q, p, (size_t)used * per * sizeof(T), cudaMemcpyDeviceToDevice);
      p = q;
    };
    move(lo_g, 1);
    move(hi_g, 1);
    move(par_g, 1);
    move(ijk_g, 3);
    move(lev_g, 1);
    move(leaf_g, 1);
    cap = nc;
    return S.err;
  };
  uint8_t* alive = S.get<uint8_t>(m);
  int32_t* pbox = S.get<int32_t>(m);
  int32_t* start = S.get<int32_t>(m);
  int32_t* incl = S.get<int32_t>(m);
  int* overflow = S.get<int>(1);
  TD_TRY(S.err);
  const int64_t zero64 = 0;
  const int32_t zero32 = 0, minus1 = -1;
  const uint8_t root_leaf = m <= t.ncrit ? 1 : 0;
  TD_TRY(cudaMemcpy(lo_g, &zero64, 8, cudaMemcpyHostToDevice));
  TD_TRY(cudaMemcpy(hi_g, &m, 8, cudaMemcpyHostToDevice));
  TD_TRY(cudaMemcpy(par_g, &minus1, 4, cudaMemcpyHostToDevice));
  TD_TRY(cudaMemset(ijk_g, 0, 24));
  TD_TRY(cudaMemcpy(lev_g, &zero32, 4, cudaMemcpyHostToDevice));
  TD_TRY(cudaMemcpy(leaf_g, &root_leaf, 1, cudaMemcpyHostToDevice));
  TD_TRY(cudaMemset(alive, root_leaf ? 0 : 1, m));
  TD_TRY(cudaMemset(pbox, 0, 4 * m));
  TD_TRY(cudaMemset(overflow, 0, sizeof(int)));
  std::vector<int64_t> lvl_off{0, 1};
  for (int lev = 1; lev <= kMaxDepth && lvl_off[lev] > lvl_off[lev - 1]; ++lev) {
    // any non-leaf box at lev - 1?  (leaf flags of that level on the host)
    std::vector<uint8_t> pl;
    TD_TRY(d2h(pl, leaf_g + lvl_off[lev - 1], lvl_off[lev] - lvl_off[lev - 1]));
    bool any = false;
    for (uint8_t v : pl) any |= v == 0;
    if (!any) break;
    level_flags_kernel<<<blocks(m), kT>>>(codes, alive, m, lev, start);
    TD_TRY(cudaGetLastError());
    TD_TRY(scan_incl(S, start, incl, m));
    int32_t nlevel = 0;
    TD_TRY(cudaMemcpy(&nlevel, incl + m - 1, 4, cudaMemcpyDeviceToHost));
    const int64_t g0 = lvl_off[lev];
    if (g0 + nlevel > cap) TD_TRY(grow(g0 + nlevel, g0));
    level_boxes_kernel<<<blocks(m), kT>>>(codes, alive, start, incl, pbox, m, lev, g0, lo_g, hi_g, par_g,
                                          ijk_g, lev_g);
    TD_TRY(cudaGetLastError());
    level_leaf_kernel<<<blocks(nlevel), kT>>>(lo_g, hi_g, g0, nlevel, lev, t.ncrit, leaf_g, overflow);
    TD_TRY(cudaGetLastError());
    level_alive_kernel<<<blocks(m), kT>>>(incl, leaf_g, m, g0, alive, pbox);
    TD_TRY(cudaGetLastError());
    lvl_off.push_back(g0 + nlevel);
  }
  int ovf = 0;
  TD_TRY(cudaMemcpy(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost));
  if (ovf)
    return fail(LB_ERR_CAPACITY, "octree depth cap 20 exceeded (pathological clustering)");
  const int nlev = (int)lvl_off.size() - 1;
  const int64_t nbox = lvl_off[nlev];
  // children, subtree sizes, preorder, ids
  int32_t* first = S.get<int32_t>(nbox);
  int32_t* nchild = S.get<int32_t>(nbox);
  int32_t* size = S.get<int32_t>(nbox);
  int32_t* pos = S.get<int32_t>(nbox);
  int32_t* nc_at = S.get<int32_t>(nbox);
  int32_t* base_at = S.get<int32_t>(nbox);
  int32_t* id = S.get<int32_t>(nbox);
  TD_TRY(S.err);
  TD_TRY(cudaMemset(nchild, 0, 4 * nbox));
  TD_TRY(cudaMemset(first, 0, 4 * nbox));
  TD_TRY(cudaMemset(pos, 0, 4 * nbox));
  for (int lev = 1; lev < nlev; ++lev) {
    const int64_t n = lvl_off[lev + 1] - lvl_off[lev];
    children_kernel<<<blocks(n), kT>>>(par_g, lvl_off[lev], n, first, nchild);
    TD_TRY(cudaGetLastError());
  }
  for (int lev = nlev - 1; lev >= 0; --lev) {
    const int64_t n = lvl_off[lev + 1] - lvl_off[lev];
    subtree_kernel<<<blocks(n), kT>>>(first, nchild, lvl_off[lev], n, size);
    TD_TRY(cudaGetLastError());
  }
  for (int lev = 0; lev < nlev - 1; ++lev) {
    const int64_t n = lvl_off[lev + 1] - lvl_off[lev];
    preorder_kernel<<<blocks(n), kT>>>(first, nchild, size, lvl_off[lev], n, pos);
    TD_TRY(cudaGetLastError());
  }
  scatter_by_pos_kernel<<<blocks(nbox), kT>>>(pos, nchild, nbox, nc_at);
  TD_TRY(cudaGetLastError());
  TD_TRY(scan_excl(S, nc_at, base_at, nbox));
  ids_kernel<<<blocks(nbox), kT>>>(pos, first, nchild, base_at, nbox, id);
  TD_TRY(cudaGetLastError());
  // sources / targets in sorted order (fmm.py:631-635)
  int64_t* is_src = S.get<int64_t>(m + 1);
  int64_t* is_tgt = S.get<int64_t>(m + 1);
  int64_t* ps = S.get<int64_t>(m + 1);
  int64_t* pt = S.get<int64_t>(m + 1);
  int64_t* src_sorted = S.get<int64_t>(t.ns);
  int64_t* tgt_sorted = S.get<int64_t>(t.nt);
  TD_TRY(S.err);
  TD_TRY(cudaMemset(is_src + m, 0, 8));
  TD_TRY(cudaMemset(is_tgt + m, 0, 8));
  src_flags_kernel<<<blocks(m), kT>>>(order, m, t.ns, is_src, is_tgt);
  TD_TRY(cudaGetLastError());
  TD_TRY(scan_excl(S, is_src, ps, m + 1));
  TD_TRY(scan_excl(S, is_tgt, pt, m + 1));
  split_kernel<<<blocks(m), kT>>>(order, ps, pt, m, t.ns, src_sorted, tgt_sorted);
  TD_TRY(cudaGetLastError());
  // per-box arrays in id order
  int32_t* level = S.get<int32_t>(nbox);
  int64_t* ijk = S.get<int64_t>(3 * nbox);
  int64_t* parent = S.get<int64_t>(nbox);
  uint8_t* leaf = S.get<uint8_t>(nbox);
  int64_t* lo = S.get<int64_t>(nbox);
  int64_t* hi = S.get<int64_t>(nbox);
  int64_t* nch = S.get<int64_t>(nbox + 1);
  int64_t* coff = S.get<int64_t>(nbox + 1);
  int64_t* srng = S.get<int64_t>(2 * nbox);
  int64_t* trng = S.get<int64_t>(2 * nbox);
  int64_t* cidx = S.get<int64_t>(nbox);
  TD_TRY(S.err);
  TD_TRY(cudaMemset(nch + nbox, 0, 8));
  by_id_kernel<<<blocks(nbox), kT>>>(id, lev_g, ijk_g, par_g, leaf_g, lo_g, hi_g, nchild, ps, pt, nbox, level,
                                     ijk, parent, leaf, lo, hi, nch, srng, trng);
  TD_TRY(cudaGetLastError());
  TD_TRY(scan_excl(S, nch, coff, nbox + 1));
  children_idx_kernel<<<blocks(nbox), kT>>>(id, first, nchild, coff, nbox, cidx);
  TD_TRY(cudaGetLastError());
  // interaction lists
  const auto l0 = std::chrono::steady_clock::now();
  t.buffer = buffer;
  const int K = (2 * buffer + 1) * (2 * buffer + 1) * (2 * buffer + 1);
  int64_t* nsrc_g = S.get<int64_t>(nbox);
  int64_t* ntgt_g = S.get<int64_t>(nbox);
  int32_t* cols = S.get<int32_t>(nbox * K);
  int32_t* ncol = S.get<int32_t>(nbox);
  int64_t* cnt = S.get<int64_t>(nbox + 1);
  int64_t* cnt2 = S.get<int64_t>(nbox + 1);
  int64_t* cnt3 = S.get<int64_t>(nbox + 1);
  TD_TRY(S.err);
  box_counts_kernel<<<blocks(nbox), kT>>>(lo_g, hi_g, ps, pt, nbox, nsrc_g, ntgt_g);
  TD_TRY(cudaGetLastError());
  const GTree T{lev_g, ijk_g, par_g, leaf_g, first, nchild, nsrc_g, ntgt_g, id, cols, ncol, K, buffer};
  TD_TRY(cudaMemcpy(cols, &zero32, 4, cudaMemcpyHostToDevice));
  {
    const int32_t one = 1;
    TD_TRY(cudaMemcpy(ncol, &one, 4, cudaMemcpyHostToDevice));
  }
  // colleagues level by level, V lengths on the way
  TD_TRY(cudaMemset(cnt, 0, 8 * (nbox + 1)));
  for (int lev = 1; lev < nlev; ++lev) {
    const int64_t n = lvl_off[lev + 1] - lvl_off[lev];
    colleagues_kernel<false><<<blocks(n), kT>>>(T, lvl_off[lev], n, cnt, nullptr, nullptr);
    TD_TRY(cudaGetLastError());
  }
  auto csr_from_counts = [&](int64_t* counts, std::vector<int64_t>& off_h, int64_t** off_d, int64_t** idx_d,
                             int64_t* total) -> cudaError_t {
    *off_d = S.get<int64_t>(nbox + 1);
    cudaError_t e = S.err;
    if (e == cudaSuccess) e = scan_excl(S, counts, *off_d, nbox + 1);
    if (e == cudaSuccess) e = d2h(off_h, *off_d, nbox + 1);
    *total = off_h.empty() ? 0 : off_h[nbox];
    *idx_d = S.get<int64_t>(*total);
    return e == cudaSuccess ? S.err : e;
  };
  int64_t *voff = nullptr, *vidx = nullptr, nvtot = 0;
  TD_TRY(csr_from_counts(cnt, t.vlist.off, &voff, &vidx, &nvtot));
  for (int lev = 1; lev < nlev; ++lev) {
    const int64_t n = lvl_off[lev + 1] - lvl_off[lev];
    colleagues_kernel<true><<<blocks(n), kT>>>(T, lvl_off[lev], n, nullptr, voff, vidx);
    TD_TRY(cudaGetLastError());
  }
  TD_TRY(d2h(t.vlist.idx, vidx, nvtot));
  TD_TRY(cudaMemset(cnt, 0, 8 * (nbox + 1)));
  colleague_rows_kernel<<<blocks(nbox), kT>>>(T, nbox, cnt, nullptr, nullptr);
  TD_TRY(cudaGetLastError());
  int64_t *coloff = nullptr, *colidx = nullptr, ncoltot = 0;
  TD_TRY(csr_from_counts(cnt, t.colleagues.off, &coloff, &colidx, &ncoltot));
  colleague_rows_kernel<<<blocks(nbox), kT>>>(T, nbox, nullptr, coloff, colidx);
  TD_TRY(cudaGetLastError());
  TD_TRY(d2h(t.colleagues.idx, colidx, ncoltot));
  // U, W, X
  TD_TRY(cudaMemset(cnt, 0, 8 * (nbox + 1)));
  TD_TRY(cudaMemset(cnt2, 0, 8 * (nbox + 1)));
  TD_TRY(cudaMemset(cnt3, 0, 8 * (nbox + 1)));
  uwx_kernel<false><<<blocks(nbox), kT>>>(T, nbox, cnt, cnt2, cnt3, nullptr, nullptr, nullptr, nullptr, nullptr,
                                           nullptr, overflow);
  TD_TRY(cudaGetLastError());
  int64_t *uoff = nullptr, *uidx = nullptr, *woff = nullptr, *widx = nullptr, *xoff = nullptr, *xidx = nullptr;
  int64_t nu = 0, nw = 0, nx = 0;
  TD_TRY(csr_from_counts(cnt, t.ulist.off, &uoff, &uidx, &nu));
  TD_TRY(csr_from_counts(cnt2, t.wlist.off, &woff, &widx, &nw));
  TD_TRY(csr_from_counts(cnt3, t.xlist.off, &xoff, &xidx, &nx));
  TD_TRY(cudaMemcpy(cnt3, xoff, 8 * (nbox + 1), cudaMemcpyDeviceToDevice));  // X cursors
  uwx_kernel<true><<<blocks(nbox), kT>>>(T, nbox, nullptr, nullptr, nullptr, uoff, woff, cnt3, uidx, widx, xidx,
                                          overflow);
  TD_TRY(cudaGetLastError());
  sort_rows_kernel<<<blocks(nbox), kT>>>(xoff, nbox, xidx);
  TD_TRY(cudaGetLastError());
  TD_TRY(cudaMemcpy(&ovf, overflow, sizeof(int), cudaMemcpyDeviceToHost));
  if (ovf) return fail(LB_ERR_CUDA, "fmm device lists: DFS stack overflow");
  TD_TRY(d2h(t.ulist.idx, uidx, nu));
  TD_TRY(d2h(t.wlist.idx, widx, nw));
  TD_TRY(d2h(t.xlist.idx, xidx, nx));
  if (lists_ms)
    *lists_ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - l0).count();
  // host copies (the lists and the apply's device state are built from them)
  TD_TRY(d2h(t.level, level, nbox));
  TD_TRY(d2h(t.ijk, ijk, 3 * nbox));
  TD_TRY(d2h(t.parent, parent, nbox));
  TD_TRY(d2h(t.is_leaf, leaf, nbox));
  TD_TRY(d2h(t.lo, lo, nbox));
  TD_TRY(d2h(t.hi, hi, nbox));
  TD_TRY(d2h(t.children.off, coff, nbox + 1));
  TD_TRY(d2h(t.children.idx, cidx, nbox - 1));
  TD_TRY(d2h(t.src_sorted, src_sorted, t.ns));
  TD_TRY(d2h(t.tgt_sorted, tgt_sorted, t.nt));
  std::vector<int64_t> sr, tr;
  TD_TRY(d2h(sr, srng, 2 * nbox));
  TD_TRY(d2h(tr, trng, 2 * nbox));
  t.codes.clear();  // the sorted keys and order stay on the device (unused on the host)
  t.order.clear();
  t.src_lo.resize(nbox);
  t.src_hi.resize(nbox);
  t.tgt_lo.resize(nbox);
  t.tgt_hi.resize(nbox);
  t.nsrc.resize(nbox);
  t.nlev = nlev;
  t.levels.assign(nlev, {});
  for (int64_t b = 0; b < nbox; ++b) {
    t.src_lo[b] = sr[2 * b];
    t.src_hi[b] = sr[2 * b + 1];
    t.tgt_lo[b] = tr[2 * b];
    t.tgt_hi[b] = tr[2 * b + 1];
    t.nsrc[b] = t.src_hi[b] - t.src_lo[b];  // a box's range holds exactly its subtree (fmm.py:636-639)
    t.levels[t.level[b]].push_back(b);
  }
  if (keep) {
    keep->release();
    keep->spos = S.release(ds);
    keep->tpos = S.release(dt);
    keep->src_sorted = S.release(src_sorted);
    keep->tgt_sorted = S.release(tgt_sorted);
    keep->v_off = S.release(voff);
    keep->v_idx = S.release(vidx);
  }
  return LB_OK;
}

}  // namespace lb
