// Native octree + interaction lists (see fmm_tree.h).  Host C++: the tree is
// plan-time work whose cost is dominated by the key sort, which the device
// path does on the GPU; the DFS numbering and the list walks are O(boxes).
#include "fmm_tree.h"

#include <algorithm>
#include <cmath>
#include <numeric>
#include <string>

#include "../../include/lapbel_b200.h"

namespace lb {

int fail(int code, const std::string& msg);

void tree_bounds(const double* spos, int64_t ns, const double* tpos, int64_t nt, double center[3],
                 double* half) {
  double lo[3] = {INFINITY, INFINITY, INFINITY}, hi[3] = {-INFINITY, -INFINITY, -INFINITY};
  auto scan = [&](const double* p, int64_t n) {
    for (int64_t i = 0; i < n; ++i)
      for (int a = 0; a < 3; ++a) {
        lo[a] = std::min(lo[a], p[3 * i + a]);
        hi[a] = std::max(hi[a], p[3 * i + a]);
      }
  };
  scan(spos, ns);
  scan(tpos, nt);
  double ext = -INFINITY;
  for (int a = 0; a < 3; ++a) {
    center[a] = 0.5 * (lo[a] + hi[a]);  // fmm.py:564
    ext = std::max(ext, hi[a] - lo[a]);
  }
  double h = 0.5 * ext;                 // fmm.py:565
  volatile double grow = 1.0 + 1e-9;    // the Python constant, rounded once
  h = h * grow;
  h = h + 1e-300;                       // fmm.py:566
  *half = h;
}

uint64_t morton_key(const double* p, const double center[3], double half) {
  // fmm.py:569-576: q = (x - (center - half)) / (2 half); cell = trunc(q 2^20)
  // clipped to [0, 2^20 - 1]; bit 3b+axis of the key = bit b of cell[axis]
  const double scale = (double)(1 << kMaxDepth);
  uint64_t code = 0;
  for (int a = 0; a < 3; ++a) {
    const double origin = center[a] - half;
    const double q = (p[a] - origin) / (2.0 * half);
    int64_t cell = (int64_t)(q * scale);
    cell = std::min<int64_t>(std::max<int64_t>(cell, 0), (1 << kMaxDepth) - 1);
    for (int b = 0; b < kMaxDepth; ++b) code |= (uint64_t)((cell >> b) & 1) << (3 * b + a);
  }
  return code;
}

double FmmTree::box_half(int64_t b) const { return half / std::ldexp(1.0, level[b]); }

void FmmTree::box_center(int64_t b, double* c) const {
  // fmm.py:642-643: (center - half) + (ijk + 0.5) * (2 * halves)
  const double hb = box_half(b);
  for (int a = 0; a < 3; ++a)
    c[a] = (center[a] - half) + ((double)ijk[3 * b + a] + 0.5) * (2.0 * hb);
}

int tree_from_sorted(FmmTree& t, std::vector<uint64_t>&& codes, std::vector<int64_t>&& order) {
  const int64_t m = (int64_t)codes.size();
  t.codes = std::move(codes);
  t.order = std::move(order);
  t.level.clear();
  t.ijk.clear();
  t.parent.clear();
  t.is_leaf.clear();
  t.lo.clear();
  t.hi.clear();
  std::vector<std::vector<int64_t>> kids;
  auto add_box = [&](int lev, int64_t x, int64_t y, int64_t z, int64_t par, int64_t lo,
                     int64_t hi) {
    const int64_t id = (int64_t)t.level.size();
    t.level.push_back(lev);
    t.ijk.push_back(x);
    t.ijk.push_back(y);
    t.ijk.push_back(z);
    t.parent.push_back(par);
    t.is_leaf.push_back(0);
    t.lo.push_back(lo);
    t.hi.push_back(hi);
    kids.emplace_back();
    if (par >= 0) kids[par].push_back(id);
    return id;
  };
  add_box(0, 0, 0, 0, -1, 0, m);
  std::vector<int64_t> stack{0};
  const uint64_t* cs = t.codes.data();
  while (!stack.empty()) {  // DFS with a LIFO stack, fmm.py:598-629
    const int64_t b = stack.back();
    stack.pop_back();
    const int64_t lo = t.lo[b], hi = t.hi[b], npts = hi - lo;
    const int lev = t.level[b];
    if (npts <= t.ncrit || lev == kMaxDepth) {
      if (lev == kMaxDepth && npts > 64 * (int64_t)t.ncrit)
        return fail(LB_ERR_CAPACITY, "octree depth cap 20 exceeded with " + std::to_string(npts) +
                                         " points in one cell (pathological clustering)");
      t.is_leaf[b] = 1;
      continue;
    }
    const int shift = 3 * (kMaxDepth - lev - 1);
    const uint64_t base = cs[lo] >> (3 * (kMaxDepth - lev));
    int64_t cuts[9];
    cuts[0] = lo;
    for (int oct = 1; oct < 8; ++oct) {
      const uint64_t key = ((base << 3) | (uint64_t)oct) << shift;
      cuts[oct] = std::lower_bound(cs + lo, cs + hi, key) - cs;
    }
    cuts[8] = hi;
    const int64_t cx = t.ijk[3 * b], cy = t.ijk[3 * b + 1], cz = t.ijk[3 * b + 2];
    for (int oct = 0; oct < 8; ++oct) {
      if (cuts[oct + 1] > cuts[oct]) {
        const int64_t id = add_box(lev + 1, 2 * cx + (oct & 1), 2 * cy + ((oct >> 1) & 1),
                                   2 * cz + ((oct >> 2) & 1), b, cuts[oct], cuts[oct + 1]);
        stack.push_back(id);
      }
    }
  }
  const int64_t nbox = t.nbox();
  t.children = Csr();
  for (int64_t b = 0; b < nbox; ++b) t.children.push_row(kids[b]);
  // sorted source / target lists and every box's range in them
  t.src_sorted.clear();
  t.tgt_sorted.clear();
  std::vector<int64_t> ps(m + 1, 0), pt(m + 1, 0);
  for (int64_t p = 0; p < m; ++p) {
    const int64_t idx = t.order[p];
    const bool is_src = idx < t.ns;
    if (is_src) t.src_sorted.push_back(idx);
    else t.tgt_sorted.push_back(idx - t.ns);
    ps[p + 1] = ps[p] + (is_src ? 1 : 0);
    pt[p + 1] = pt[p] + (is_src ? 0 : 1);
  }
  t.src_lo.resize(nbox);
  t.src_hi.resize(nbox);
  t.tgt_lo.resize(nbox);
  t.tgt_hi.resize(nbox);
  t.nsrc.assign(nbox, 0);
  int maxlev = 0;
  for (int64_t b = 0; b < nbox; ++b) {
    t.src_lo[b] = ps[t.lo[b]];
    t.src_hi[b] = ps[t.hi[b]];
    t.tgt_lo[b] = pt[t.lo[b]];
    t.tgt_hi[b] = pt[t.hi[b]];
    if (t.is_leaf[b]) t.nsrc[b] = t.src_hi[b] - t.src_lo[b];
    maxlev = std::max(maxlev, (int)t.level[b]);
  }
  for (int64_t b = nbox - 1; b > 0; --b) t.nsrc[t.parent[b]] += t.nsrc[b];  // fmm.py:638-639
  t.nlev = maxlev + 1;
  t.levels.assign(t.nlev, {});
  for (int64_t b = 0; b < nbox; ++b) t.levels[t.level[b]].push_back(b);
  return LB_OK;
}

int tree_build_host(FmmTree& t, const double* spos, int64_t ns, const double* tpos, int64_t nt,
                    int ncrit) {
  t.ns = ns;
  t.nt = nt;
  t.ncrit = ncrit;
  tree_bounds(spos, ns, tpos, nt, t.center, &t.half);
  const int64_t m = ns + nt;
  std::vector<uint64_t> code(m);
  for (int64_t i = 0; i < m; ++i)
    code[i] = morton_key(i < ns ? spos + 3 * i : tpos + 3 * (i - ns), t.center, t.half);
  std::vector<int64_t> order(m);
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](int64_t a, int64_t b) { return code[a] < code[b]; });  // fmm.py:577
  std::vector<uint64_t> sorted(m);
  for (int64_t p = 0; p < m; ++p) sorted[p] = code[order[p]];
  return tree_from_sorted(t, std::move(sorted), std::move(order));
}

// fmm.py:650-659
static bool near_boxes(const FmmTree& t, int64_t a, int64_t b, int buffer) {
  const int la = t.level[a], lb2 = t.level[b];
  const int lf = std::max(la, lb2);
  const int64_t sa = (int64_t)1 << (lf - la), sb = (int64_t)1 << (lf - lb2);
  const int64_t m = std::min(sa, sb) * buffer;
  for (int k = 0; k < 3; ++k) {
    const int64_t alo = t.ijk[3 * a + k] * sa, blo = t.ijk[3 * b + k] * sb;
    const int64_t gap = std::max(blo - (alo + sa), alo - (blo + sb));
    if (!(gap < m)) return false;
  }
  return true;
}

// Lists in flat arrays, every pass parallel over boxes (OpenMP) and every
// list in the reference's order: the count and the fill of a box run the
// same walk, so placement depends on the box alone.
void tree_lists(FmmTree& t, int buffer) {
  t.buffer = buffer;
  const int64_t nbox = t.nbox();
  const int K = (2 * buffer + 1) * (2 * buffer + 1) * (2 * buffer + 1);  // colleagues per box, max
  std::vector<int32_t> colf((size_t)nbox * K), ncol(nbox, 0);
  std::vector<int64_t> nv(nbox, 0);
  colf[0] = 0;
  ncol[0] = 1;
  const int64_t* ijk = t.ijk.data();
  auto cheb = [&](int64_t a, int64_t b) {
    return std::max({std::llabs(ijk[3 * a] - ijk[3 * b]), std::llabs(ijk[3 * a + 1] - ijk[3 * b + 1]),
                     std::llabs(ijk[3 * a + 2] - ijk[3 * b + 2])});
  };
  // colleagues and V, level by level (fmm.py:669-679): children of the
  // parent's colleagues, in the parent's colleague order then octant order
  auto walk_cv = [&](int64_t b, auto&& on_col, auto&& on_v) {
    const int64_t p = t.parent[b];
    for (int q = 0; q < ncol[p]; ++q) {
      const int64_t pc = colf[(size_t)p * K + q];
      const int64_t* ch = t.children.row(pc);
      for (int64_t r = 0; r < t.children.size(pc); ++r) {
        const int64_t c = ch[r];
        if (cheb(c, b) <= buffer) on_col(c);
        else if (t.nsrc[c] > 0) on_v(c);
      }
    }
  };
  for (int lev = 1; lev < t.nlev; ++lev) {
    const std::vector<int64_t>& L = t.levels[lev];
#pragma omp parallel for schedule(dynamic, 512)
    for (int64_t i = 0; i < (int64_t)L.size(); ++i) {
      const int64_t b = L[i];
      int nc = 0;
      int64_t cv = 0;
      int32_t* dst = &colf[(size_t)b * K];
      walk_cv(b, [&](int64_t c) { dst[nc++] = (int32_t)c; }, [&](int64_t) { ++cv; });
      ncol[b] = nc;
      nv[b] = cv;
    }
  }
  auto scan = [&](const std::vector<int64_t>& cnt, Csr& out) {
    out.off.assign(nbox + 1, 0);
    for (int64_t b = 0; b < nbox; ++b) out.off[b + 1] = out.off[b] + cnt[b];
    out.idx.assign(out.off[nbox], 0);
  };
  {
    std::vector<int64_t> nc64(ncol.begin(), ncol.end());
    scan(nc64, t.colleagues);
  }
  scan(nv, t.vlist);
#pragma omp parallel for schedule(dynamic, 512)
  for (int64_t b = 0; b < nbox; ++b) {
    int64_t* c = &t.colleagues.idx[t.colleagues.off[b]];
    for (int q = 0; q < ncol[b]; ++q) c[q] = colf[(size_t)b * K + q];
    if (b == 0) continue;
    int64_t* v = &t.vlist.idx[t.vlist.off[b]];
    int64_t n = 0;
    walk_cv(b, [](int64_t) {}, [&](int64_t k) { v[n++] = k; });
  }
  // U, W, X for non-empty leaves in ascending id (fmm.py:684-714).  The
  // reference dedupes the ancestor walk with a set; colleagues of an
  // ancestor a are boxes of a's level, so no box can repeat there.
  auto walk_uwx = [&](int64_t b, std::vector<int64_t>& stack, auto&& on_u, auto&& on_w, auto&& on_x) {
    const bool has_src = t.src_hi[b] > t.src_lo[b];
    for (int64_t a = b; a != -1; a = t.parent[a])
      for (int q = 0; q < ncol[a]; ++q) {
        const int64_t c = colf[(size_t)a * K + q];
        if (t.is_leaf[c] && c != b && near_boxes(t, b, c, buffer)) on_u(c);
      }
    on_u(b);
    stack.clear();
    for (int q = 0; q < ncol[b]; ++q) {
      const int64_t c = colf[(size_t)b * K + q];
      if (!t.is_leaf[c]) stack.push_back(c);
    }
    while (!stack.empty()) {
      const int64_t c = stack.back();
      stack.pop_back();
      const int64_t* ch = t.children.row(c);
      for (int64_t q = 0; q < t.children.size(c); ++q) {
        const int64_t k = ch[q];
        if (near_boxes(t, b, k, buffer)) {
          if (t.is_leaf[k]) on_u(k);
          else stack.push_back(k);
        } else {
          if (t.nsrc[k] > 0) on_w(k);
          if (has_src) on_x(k);
        }
      }
    }
  };
  auto active = [&](int64_t b) {
    return t.is_leaf[b] && (t.tgt_hi[b] > t.tgt_lo[b] || t.src_hi[b] > t.src_lo[b]);
  };
  std::vector<int64_t> nu(nbox, 0), nw(nbox, 0), nx(nbox, 0);
#pragma omp parallel
  {
    std::vector<int64_t> stack;
#pragma omp for schedule(dynamic, 256)
    for (int64_t b = 0; b < nbox; ++b) {
      if (!active(b)) continue;
      int64_t cu = 0, cw = 0;
      walk_uwx(b, stack, [&](int64_t) { ++cu; }, [&](int64_t) { ++cw; }, [&](int64_t k) {
#pragma omp atomic
        ++nx[k];
      });
      nu[b] = cu;
      nw[b] = cw;
    }
  }
  scan(nu, t.ulist);
  scan(nw, t.wlist);
  scan(nx, t.xlist);
  std::vector<int64_t> xcur(t.xlist.off.begin(), t.xlist.off.end() - 1);
#pragma omp parallel
  {
    std::vector<int64_t> stack;
#pragma omp for schedule(dynamic, 256)
    for (int64_t b = 0; b < nbox; ++b) {
      if (!active(b)) continue;
      int64_t* u = &t.ulist.idx[t.ulist.off[b]];
      int64_t* w = &t.wlist.idx[t.wlist.off[b]];
      int64_t cu = 0, cw = 0;
      walk_uwx(b, stack, [&](int64_t k) { u[cu++] = k; }, [&](int64_t k) { w[cw++] = k; },
               [&](int64_t k) {
                 int64_t pos;
#pragma omp atomic capture
                 pos = xcur[k]++;
                 t.xlist.idx[pos] = b;
               });
    }
  }
  // X[k] lists its sources in ascending leaf id, as the reference's loop order
#pragma omp parallel for schedule(dynamic, 512)
  for (int64_t k = 0; k < nbox; ++k)
    std::sort(t.xlist.idx.begin() + t.xlist.off[k], t.xlist.idx.begin() + t.xlist.off[k + 1]);
}

}  // namespace lb
