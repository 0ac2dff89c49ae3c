// Adaptive octree and interaction lists of the reference FMM plan
// (fmm.py:539-715), rebuilt natively.  Integer structure is bit-exact with
// `_build_tree` / `_build_lists`: same Morton keys, same stable order, same
// DFS-LIFO box numbering, same list contents and order.
#pragma once

#include <stdint.h>

#include <vector>

namespace lb {

constexpr int kMaxDepth = 20;  // fmm.py:539

struct Csr {
  std::vector<int64_t> off{0};
  std::vector<int64_t> idx;
  void push_row(const std::vector<int64_t>& r) {
    idx.insert(idx.end(), r.begin(), r.end());
    off.push_back((int64_t)idx.size());
  }
  int64_t size(int64_t b) const { return off[b + 1] - off[b]; }
  const int64_t* row(int64_t b) const { return idx.data() + off[b]; }
};

struct FmmTree {
  int64_t ns = 0, nt = 0;
  int ncrit = 0, buffer = 1;
  double center[3] = {0, 0, 0};
  double half = 0;
  int nlev = 0;
  // per box, indexed by the reference's box id
  std::vector<int32_t> level;
  std::vector<int64_t> ijk;  // 3 per box
  std::vector<int64_t> parent;
  Csr children;              // ascending octant order
  std::vector<uint8_t> is_leaf;
  std::vector<int64_t> lo, hi;  // point range in the sorted order
  std::vector<int64_t> nsrc;    // subtree source count (fmm.py:636-639)
  std::vector<int64_t> order;   // sorted position -> index into vstack([spos, tpos])
  std::vector<uint64_t> codes;  // sorted Morton codes
  // sources / targets in sorted order, and every box's contiguous range in them
  std::vector<int64_t> src_sorted, tgt_sorted;  // original source / target indices
  std::vector<int64_t> src_lo, src_hi, tgt_lo, tgt_hi;
  std::vector<std::vector<int64_t>> levels;  // box ids per level, ascending
  // lists (fmm.py:662-715)
  Csr colleagues, vlist, ulist, wlist, xlist;

  int64_t nbox() const { return (int64_t)level.size(); }
  double box_half(int64_t b) const;
  void box_center(int64_t b, double* c) const;
};

// Morton code of one point exactly as fmm.py:562-576 (host arithmetic).
void tree_bounds(const double* spos, int64_t ns, const double* tpos, int64_t nt,
                 double center[3], double* half);

// Build the tree from codes already sorted (stable) with their original
// indices; returns LB_OK or LB_ERR_CAPACITY (fmm.py:605-609).
int tree_from_sorted(FmmTree& t, std::vector<uint64_t>&& codes, std::vector<int64_t>&& order);

// Host path: keys + std::stable_sort.  The device path (fmm_plan.cu) computes
// the same keys on the GPU and radix-sorts them.
int tree_build_host(FmmTree& t, const double* spos, int64_t ns, const double* tpos, int64_t nt,
                    int ncrit);

void tree_lists(FmmTree& t, int buffer);

uint64_t morton_key(const double* p, const double center[3], double half);

}  // namespace lb
