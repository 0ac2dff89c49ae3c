// The FMM plan handle: octree + lists (fmm_tree.cpp), device-side Morton
// keys and radix sort, tree export for the bit-exact checks, and (fmm_apply.cu)
// the device passes.  FmmPlan.__init__ equivalent (fmm.py:729-748).
#include <cub/cub.cuh>

#include <chrono>
#include <cstring>
#include <string>

#include "fmm_plan.h"
#include "lb_common.cuh"

using namespace lb;

extern "C" {

int lb_fmm_plan_create(const double* spos, int64_t ns, const double* tpos, int64_t nt, int ncrit,
                       int buffer, int flags, lb_fmm_plan** out) {
  if (!out) return fail(LB_ERR_ARG, "lb_fmm_plan_create: null output");
  *out = nullptr;
  if (ns < 0 || nt < 0 || ns + nt == 0) return fail(LB_ERR_SHAPE, "lb_fmm_plan_create: no points");
  if (ncrit < 1 || buffer < 1) return fail(LB_ERR_ARG, "lb_fmm_plan_create: ncrit, buffer >= 1");
  if ((ns && !spos) || (nt && !tpos)) return fail(LB_ERR_ARG, "lb_fmm_plan_create: null positions");
  lb_fmm_plan* p = new lb_fmm_plan();
  FmmTree& t = p->tree;
  t.ns = ns;
  t.nt = nt;
  t.ncrit = ncrit;
  int rc;
  using clk = std::chrono::steady_clock;
  auto ms = [](clk::time_point a, clk::time_point b) {
    return std::chrono::duration<double, std::milli>(b - a).count();
  };
  const auto c0 = clk::now();
  auto c1 = c0;
  double dev_lists_ms = -1;
  if (flags & LB_FMM_DEVICE_SORT) {
    rc = tree_build_device(t, spos, tpos, buffer, &dev_lists_ms, &p->tdev);  // fmm_tree_dev.cu
    c1 = clk::now();
  } else {
    rc = tree_build_host(t, spos, ns, tpos, nt, ncrit);
  }
  if (rc != LB_OK) {
    p->tdev.release();
    delete p;
    return rc;
  }
  const auto c2 = clk::now();
  if (dev_lists_ms < 0) tree_lists(t, buffer);
  const auto c3 = clk::now();
  p->setup_ms[0] = ms(c0, c1);
  p->setup_ms[1] = ms(c1, c2);
  p->setup_ms[2] = ms(c2, c3);
  if (dev_lists_ms >= 0) {  // the device build timed its lists inside the first interval
    p->setup_ms[0] -= dev_lists_ms;
    p->setup_ms[2] = dev_lists_ms;
  }
  p->spos.assign(spos, spos + 3 * ns);
  p->tpos.assign(tpos, tpos + 3 * nt);
  *out = p;
  return LB_OK;
}

int lb_fmm_plan_destroy(lb_fmm_plan* p) {
  if (!p) return LB_OK;
  fmm_release_device(p);
  p->tdev.release();
  delete p;
  return LB_OK;
}

int lb_fmm_setup_times(const lb_fmm_plan* p, double* out) {
  if (!p || !out) return fail(LB_ERR_ARG, "lb_fmm_setup_times: null argument");
  double tot = 0;
  for (int i = 0; i < 4; ++i) tot += (out[i] = p->setup_ms[i]);
  out[4] = tot;
  return LB_OK;
}

int lb_fmm_plan_info(const lb_fmm_plan* p, int64_t* sizes, double* geom) {
  if (!p) return fail(LB_ERR_ARG, "lb_fmm_plan_info: null plan");
  const FmmTree& t = p->tree;
  if (sizes) {
    sizes[0] = t.nbox();
    sizes[1] = t.nlev;
    sizes[2] = t.ns;
    sizes[3] = t.nt;
    sizes[4] = (int64_t)t.children.idx.size();
    sizes[5] = (int64_t)t.colleagues.idx.size();
    sizes[6] = (int64_t)t.vlist.idx.size();
    sizes[7] = (int64_t)t.ulist.idx.size();
    sizes[8] = (int64_t)t.wlist.idx.size();
    sizes[9] = (int64_t)t.xlist.idx.size();
  }
  if (geom) {
    geom[0] = t.center[0];
    geom[1] = t.center[1];
    geom[2] = t.center[2];
    geom[3] = t.half;
  }
  return LB_OK;
}

int lb_fmm_plan_export(const lb_fmm_plan* p, int what, int64_t* dst) {
  if (!p || !dst) return fail(LB_ERR_ARG, "lb_fmm_plan_export: null argument");
  const FmmTree& t = p->tree;
  const int64_t nb = t.nbox();
  auto put = [&](const std::vector<int64_t>& v) { std::memcpy(dst, v.data(), v.size() * 8); };
  switch (what) {
    case LB_TREE_LEVEL: for (int64_t b = 0; b < nb; ++b) dst[b] = t.level[b]; break;
    case LB_TREE_IJK: put(t.ijk); break;
    case LB_TREE_PARENT: put(t.parent); break;
    case LB_TREE_IS_LEAF: for (int64_t b = 0; b < nb; ++b) dst[b] = t.is_leaf[b]; break;
    case LB_TREE_NSRC: put(t.nsrc); break;
    case LB_TREE_CHILDREN_OFF: put(t.children.off); break;
    case LB_TREE_CHILDREN: put(t.children.idx); break;
    case LB_TREE_SRC_SORTED: put(t.src_sorted); break;
    case LB_TREE_TGT_SORTED: put(t.tgt_sorted); break;
    case LB_TREE_SRC_LO: put(t.src_lo); break;
    case LB_TREE_SRC_HI: put(t.src_hi); break;
    case LB_TREE_TGT_LO: put(t.tgt_lo); break;
    case LB_TREE_TGT_HI: put(t.tgt_hi); break;
    case LB_TREE_COLLEAGUES_OFF: put(t.colleagues.off); break;
    case LB_TREE_COLLEAGUES: put(t.colleagues.idx); break;
    case LB_TREE_V_OFF: put(t.vlist.off); break;
    case LB_TREE_V: put(t.vlist.idx); break;
    case LB_TREE_U_OFF: put(t.ulist.off); break;
    case LB_TREE_U: put(t.ulist.idx); break;
    case LB_TREE_W_OFF: put(t.wlist.off); break;
    case LB_TREE_W: put(t.wlist.idx); break;
    case LB_TREE_X_OFF: put(t.xlist.off); break;
    case LB_TREE_X: put(t.xlist.idx); break;
    default: return fail(LB_ERR_ARG, "lb_fmm_plan_export: unknown array");
  }
  return LB_OK;
}

}  // extern "C"
