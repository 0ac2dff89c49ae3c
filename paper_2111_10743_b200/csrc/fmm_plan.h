// lb_fmm_plan: the device FmmPlan (fmm.py:722-990).
#pragma once

#include <cuda_runtime.h>

#include <vector>

#include "../../include/lapbel_b200.h"
#include "fmm_tree.h"

namespace lb {

// device copy of everything apply() needs, built lazily on the first apply
struct FmmDevice {
  bool ready = false;
  int nd_alloc = 0;
  // geometry, sorted order
  double *spos = nullptr, *tpos = nullptr;   // sorted positions (ns,3) (nt,3)
  int64_t *src_sorted = nullptr, *tgt_sorted = nullptr;
  // per box, SLOT order (levels concatenated)
  double* bctr = nullptr;    // (nbox,3)
  double* bhalf = nullptr;   // (nbox)
  int64_t *bsrc = nullptr, *btgt = nullptr;  // (nbox,2) ranges
  // operators
  double *pts = nullptr;     // unit points (nrep,3): cube-surface lattice or Chebyshev grid
  double *pinv_up = nullptr, *pinv_dn = nullptr;
  double *m2m = nullptr, *l2l = nullptr;     // surface: 8 (nrep,nrep); grid: 2 (n,n) 1-D factors
  double *canon = nullptr;                   // (ncanon, nrep, nrep)
  int32_t *perm = nullptr, *perm_inv = nullptr;  // (noff, nrep)
  double* vinv = nullptr;                    // grid: (n,n) Chebyshev Vandermonde inverse
  // index lists (slots)
  int64_t* p2m_leaves = nullptr;             // source leaves
  int64_t n_p2m = 0;
  // m2m / l2l groups: per (level, octant) [child slot, parent slot] pairs
  int64_t *up_child = nullptr, *up_parent = nullptr;
  std::vector<int64_t> up_off;               // 8 * nlev + 1 host offsets
  int64_t *dn_child = nullptr, *dn_parent = nullptr;
  std::vector<int64_t> dn_off;
  int64_t* dn_off_dev = nullptr;             // device copy (per-octant batches of the L2L)
  int64_t* up_off_dev = nullptr;             // device copy (per-octant batches of the M2M)
  // surface M2M per level: parents (slots) with the positions of their 8
  // children in the level's child list, octant order (-1 = none), levels
  // concatenated; up_par_off: host offsets
  int64_t *up_par = nullptr, *up_child8 = nullptr;
  std::vector<int64_t> up_par_off;
  double *m2m_oct = nullptr, *l2l_oct = nullptr;  // surface operators in octant order
  // m2l: per canonical key, pairs sorted by target
  int64_t *v_src = nullptr, *v_tgt_pair_off = nullptr, *v_tgts = nullptr;
  int32_t* v_off_idx = nullptr;
  double* v_scale = nullptr;                 // 1/h of the pair's level
  std::vector<int64_t> v_key_pair_off;       // per key: pair range (host)
  std::vector<int64_t> v_key_tgt_off;        // per key: unique-target range (host)
  int64_t max_key_pairs = 0;
  // X list
  int64_t *x_boxes = nullptr, *x_off = nullptr, *x_leaves = nullptr;
  int64_t n_x = 0;
  // leaf stage
  int64_t *t_leaves = nullptr, *u_off = nullptr, *u_list = nullptr, *w_off = nullptr, *w_list = nullptr;
  int64_t n_tleaf = 0;
  // leaf work items: (target-leaf index, virtual source range [vb, ve),
  // partial offset or -1 for a leaf done by one item); heavy leaves are split
  // so no block carries more than ~2^20 pairs (load balance, not arithmetic)
  int64_t* leaf_items = nullptr;             // (n_items, 4)
  int64_t n_items = 0;
  int64_t *split_leaf = nullptr, *split_item_off = nullptr;  // split leaves, their item ranges
  int64_t n_split = 0, part_doubles = 0;     // partial slots (targets x items) of split leaves
  int64_t* leaf_item_slot = nullptr;        // per item: first partial target slot, or -1
  int64_t* leaf_order = nullptr;            // launch order of the items (heaviest first)
  double* leaf_part = nullptr;
  int64_t leaf_part_cap = 0, part_width = -1;
  // work arrays (per nd)
  double *cs = nullptr, *vs = nullptr;       // sorted charges (nd,ns), dipoles (nd,ns,3)
  uint8_t* src_own = nullptr;                // owned-source flags, sorted order (source range set)
  double *cs_own = nullptr, *vs_own = nullptr;  // the P2M's masked copies
  double *up = nullptr, *dc = nullptr, *loc = nullptr;  // (nbox, nd, nrep) slot order
  double *tmpA = nullptr, *tmpB = nullptr;   // GEMM staging
  int64_t tmp_cols = 0;
  // outputs in sorted target order (nd, nt, 10) before the scatter
  double* tout = nullptr;
  // projected leaf stage (fmm_apply_a3proj): target normals in sorted order
  // (nt, 3) and the four projections per target (nt, 4)
  double *tnrm = nullptr, *tproj = nullptr, *snrm = nullptr;
  int64_t* btgt_oct = nullptr;               // octant (x | y<<1 | z<<2) of every slot
  std::vector<int64_t> level_slot_off;       // slot range of every level
  std::vector<uint8_t> level_loc;            // per level: any owned box with a nonzero local expansion
  std::vector<int64_t> v_tpoff_host;         // host copy of v_tgt_pair_off
  // emulated-fp64 M2L on the tensor cores (ozaki.cuh), built on first use
  int oz_S = 0;                              // slices the A packs were built for
  uint8_t* oz_a = nullptr;                   // (ncanon, MT, KC, S, 4096) int8 slices
  double* oz_rs = nullptr;                   // (ncanon, MT*128) row scales
  uint8_t* oz_b = nullptr;                   // column slices of one M2L chunk
  double* oz_cs = nullptr;                   // column scales of one M2L chunk
  int64_t oz_cols = 0;                       // column capacity of oz_b / oz_cs
  // low-rank M2L (lb_fmm_plan_set_m2l_factors): per canonical key K = A B,
  // A (nrep, r_k) and B (r_k, nrep) row-major, packed; staging (r_max, cols)
  double *lr_a = nullptr, *lr_b = nullptr, *lr_t = nullptr;
  int64_t lr_t_cap = 0;
  // fused low-rank M2L (m2l_fused.cuh): B_k with its columns permuted per
  // lattice offset (lr_bp, r_k x nrep per offset at lo_aoff), every key's
  // pairs re-ordered by offset for the first factor (source slot, T column,
  // 1/h; batch boundaries lo_boff per key from lo_key_batch), and the
  // per-density-count units of whole target groups for the second
  bool lo_ready = false;
  double* lr_bp = nullptr;
  int64_t *lo_src = nullptr, *lo_tcol = nullptr, *lo_boff = nullptr, *lo_aoff = nullptr;
  double* lo_scale = nullptr;
  std::vector<int64_t> lo_key_batch, lo_key_maxgrp;    // per key: first batch entry, largest batch
  // all keys' first factors in ONE launch: batch boundaries (no duplicates),
  // factor offsets, ranks, T bases (x nd) per batch; host T base per key
  int64_t *lo_gboff = nullptr, *lo_gaoff = nullptr, *lo_gyoff = nullptr;
  int32_t *lo_gm = nullptr;
  int64_t lo_gbatch = 0, lo_gmaxgrp = 0, lo_gb0 = 0;
  int lo_rmax = 0;
  std::vector<int64_t> lo_tbase1;                      // per key: sum of pairs x r over earlier keys
  // per density count nd (1..4): units (2 x int64 target-group ranges) and
  // each key's first unit; built once per nd, so an apply never allocates
  int64_t* lo_units[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  std::vector<int64_t> lo_key_units[5];
  // fused second factor: per-unit key, batches of units (first unit / first group per batch, + end),
  // per-key table, partial-sum scratch, and every target's groups in key order for the reduction
  int32_t* lo_unit_key[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  std::vector<int64_t> lo_batch_off[5], lo_batch_grp[5];
  int64_t* lo_keytab = nullptr;
  double* lo_part = nullptr;
  int64_t lo_part_cap = 0;
  int64_t *lo_rt_tgt = nullptr, *lo_rt_off = nullptr, *lo_rt_grp = nullptr;
  int64_t lo_rt_n = 0;
  // the first factor's flat (batch, column tile) list per nd (m2l_first.cuh)
  int32_t* lo_tiles[5] = {nullptr, nullptr, nullptr, nullptr, nullptr};
  int64_t lo_ntiles[5] = {0, 0, 0, 0, 0};
  double* lr_ap = nullptr;      // A_k in DMMA fragment order (m2lf::pack_a), key k at lr_ap_off[k]
  std::vector<int64_t> lr_ap_off;
  // closed-form M2L permutations (m2lf::fit_symmetries): per offset (A, B, C, D), per point its
  // lattice coordinates, lattice index -> expansion index; lo_aff == nullptr: table lookups
  bool lo_fit_done = false;
  int32_t* lo_aff = nullptr;
  uint32_t* lo_coords = nullptr;
  uint16_t* lo_lut = nullptr;
  int lo_lut_n = 0;
  double* lo_carry = nullptr;   // m2l_fused.cuh: carry pool (lo_carry_slots x kMaxNd x nrep)
  unsigned* lo_carry_flag = nullptr;
  int lo_carry_slots = 0;
  std::vector<int32_t> lo_gm_host;
  std::vector<int64_t> lo_gb_host;
};

// device arrays kept from the device tree build (fmm_tree_dev.cu): the
// apply's device state is gathered from them instead of re-uploaded
struct TreeDev {
  double *spos = nullptr, *tpos = nullptr;         // original order
  int64_t *src_sorted = nullptr, *tgt_sorted = nullptr;
  int64_t *v_off = nullptr, *v_idx = nullptr;      // V list (by box id)
  void release() {
    cudaFree(spos); cudaFree(tpos); cudaFree(src_sorted); cudaFree(tgt_sorted);
    cudaFree(v_off); cudaFree(v_idx);
    *this = TreeDev();
  }
};

}  // namespace lb

struct lb_fmm_plan {
  lb::FmmTree tree;
  std::vector<double> spos, tpos;  // original order (host)
  // operators (host copies, set by lb_fmm_plan_set_operators)
  int rep = -1;                    // 0 surface, 1 grid
  int m = 0;                       // surface lattice size / Chebyshev order
  int nrep = 0;
  std::vector<double> pts, pinv_up, pinv_dn, m2m, l2l, canon, vinv, x1;
  std::vector<int32_t> off_key, off_perm;   // per offset index
  std::vector<int32_t> off_vec;             // (noff, 3) lattice offsets
  int ncanon = 0, noff = 0;
  double ue_scale = 1.05, uc_scale = 2.85, dc_scale = 1.05, de_scale = 2.85;
  lb::FmmDevice dev;
  lb::TreeDev tdev;                         // device tree build leftovers (empty on the host path)
  std::vector<int64_t> slot_of, id_of;      // box id <-> level-major slot
  std::vector<double> stage_ms;             // last apply's per-stage device times
  double setup_ms[4] = {0, 0, 0, 0};        // keys+sort, tree, lists, device state (host ms)
  bool timing = false;
  int64_t own_t0 = 0, own_t1 = -1;          // owned targets [t0, t1) (original order); t1 < 0: all
  int64_t own_s0 = 0, own_s1 = -1;          // owned sources [s0, s1) of the upward pass; s1 < 0: all
  lb_fmm_upward_hook up_hook = nullptr;     // sums the ranks' partial upward expansions
  void* up_hook_user = nullptr;
  int xw_direct = 0;                        // 1: cheap X / W entries evaluated directly (lb_fmm_plan_set_xw)
  int m2l_slices = 0;                       // 0: fp64 DGEMM M2L; 3..8: tcgen05 int8 slices;
                                            // -1: low-rank factors (fp64 DGEMM pair)
  std::vector<int32_t> lr_rank;             // per canonical key
  std::vector<int64_t> lr_off;              // packed offsets (ncanon + 1), in doubles per factor / nrep
  std::vector<double> lr_a_host, lr_b_host;
};

namespace lb {
void fmm_release_device(lb_fmm_plan* p);
// Device path (fmm_tree_dev.cu): keys, radix sort, boxes, the reference
// numbering and the interaction lists on the GPU; fills everything
// tree_from_sorted + tree_lists do except the sorted codes / order.
// lists_ms (optional) receives the lists' share; keep (optional) receives
// device copies of the positions, sorted index lists and the V list.
int tree_build_device(FmmTree& t, const double* spos, const double* tpos, int buffer, double* lists_ms,
                      TreeDev* keep);
// The two-density A3 call (charges (2, ns): X = c0, B = c1; dipoles (2, ns, 3):
// X only, = -c1 n_s) at level 2 with a PROJECTED leaf stage: besides
// pot/grad/hess of the grid L2T part (zero in surface mode), proj (3, nt)
// receives, in reference target order, the leaf stage's -n.grad X + n.H_B.n
// (in the accurate Kspp form, source normals snrm (ns, 3)), pot B and
// n.grad B, with n the target normals tnrm (nt, 3).  The caller adds the same
// projections of pot/grad/hess.
int fmm_apply_a3proj(lb_fmm_plan* P, const double* charges, const double* dipoles,
                     const double* tnrm, const double* snrm, double* pot, double* grad, double* hess,
                     double* proj, cudaStream_t st);
}
