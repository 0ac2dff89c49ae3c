// Direct fp64 pairwise sums of the 1/r kernel (charges and dipoles; pot,
// grad, hess) — the B200 replacement for evaluate_direct (fmm.py:130-222)
// and the numba grouped_direct (_pointsum.py:19-114).
//
// Design:
//   * sources are repacked once per call into a padded AoS record
//     [x y z | c_l | v_l.x v_l.y v_l.z ...] (16-byte aligned) so one tile of
//     TS records streams into shared memory with 128-bit loads and every
//     thread reads each record as a warp-wide broadcast;
//   * each thread owns TPT targets and keeps all accumulators in registers;
//   * 1/r: MUFU.RSQ64H seed + one 2nd-order fp64 refinement (lb_common.cuh);
//   * the sweep is decomposed stream-K (opfar.cuh): one persistent wave of
//     CTAs takes equal shares of the (target tile x source tile) units, so
//     small problems still fill the 148 SMs; per-(tile, CTA) partials are
//     reduced in a fixed order (deterministic, no fp64 atomics) by a finalize
//     kernel that also scatters into the reference layout (pot (nd,Nt),
//     grad (nd,Nt,3), hess (nd,Nt,3,3)).
#include <algorithm>
#include <string>
#include <vector>

#include "lb_common.cuh"
#include "opfar.cuh"
#include "p2p_core.cuh"

namespace lb {

// ---------------------------------------------------------------------------
// source packing

template <int NDC, bool HC, bool HD>
__global__ void pack_sources_kernel(const double* __restrict__ pos, int64_t ns, int64_t ns_pad,
                                    const double* __restrict__ charges,
                                    const double* __restrict__ dipoles, int64_t ns_total_stride,
                                    int d0, uint32_t cmask, uint32_t dmask,
                                    double* __restrict__ out) {
  using L = SrcLayout<NDC, HC, HD>;
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns_pad) return;
  double* rec = out + i * L::stride;
  if (i >= ns) {
#pragma unroll
    for (int k = 0; k < L::stride; ++k) rec[k] = 0.0;
    return;
  }
  rec[0] = pos[3 * i + 0];
  rec[1] = pos[3 * i + 1];
  rec[2] = pos[3 * i + 2];
  int o = 3;
#pragma unroll
  for (int l = 0; l < NDC; ++l) {
    const int d = d0 + l;
    if (HC) rec[o++] = ((cmask >> d) & 1u) && charges ? charges[(int64_t)d * ns_total_stride + i] : 0.0;
    if (HD) {
      const bool on = ((dmask >> d) & 1u) && dipoles;
      const double* v = dipoles + ((int64_t)d * ns_total_stride + i) * 3;
      rec[o++] = on ? v[0] : 0.0;
      rec[o++] = on ? v[1] : 0.0;
      rec[o++] = on ? v[2] : 0.0;
    }
  }
  for (; o < L::stride; ++o) rec[o] = 0.0;
}

// ---------------------------------------------------------------------------
// grouped variant: one block per group, loops over its targets and sources

template <int NDC, bool HC, bool HD, int LEVEL, int BT, int TS>
__global__ void __launch_bounds__(BT) p2p_grouped_kernel(
    const double* __restrict__ t_xyz, const int64_t* __restrict__ t_out,
    const int64_t* __restrict__ t_off, const double* __restrict__ pack,
    const int64_t* __restrict__ s_off, int64_t ntargets, int d0, int level_out,
    double* __restrict__ pot, double* __restrict__ grad, double* __restrict__ hess) {
  using L = SrcLayout<NDC, HC, HD>;
  constexpr int S = L::stride;
  constexpr int NC = ncomp(LEVEL);
  constexpr int NA = NDC * NC;
  __shared__ __align__(16) double sh[TS * S];
  const int64_t g = blockIdx.x;
  const int64_t tb = t_off[g], te = t_off[g + 1];
  const int64_t sb = s_off[g], se = s_off[g + 1];
  if (tb >= te || sb >= se) return;
  for (int64_t t0 = tb; t0 < te; t0 += BT) {
    const int64_t t = t0 + threadIdx.x;
    const bool in = t < te;
    const double tx = in ? t_xyz[3 * t + 0] : 0.0;
    const double ty = in ? t_xyz[3 * t + 1] : 0.0;
    const double tz = in ? t_xyz[3 * t + 2] : 0.0;
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    for (int64_t s0 = sb; s0 < se; s0 += TS) {
      const int n = (int)min((int64_t)TS, se - s0);
      __syncthreads();
      for (int k = threadIdx.x; k < n * S; k += BT) sh[k] = pack[s0 * S + k];
      __syncthreads();
      for (int k = 0; k < n; ++k) pair_generic<NDC, HC, HD, LEVEL>(tx, ty, tz, sh + k * S, acc);
    }
    if (in) {
      const int64_t r = t_out[t];
#pragma unroll
      for (int l = 0; l < NDC; ++l) {
        const double* a = acc + l * NC;
        const int64_t row = (int64_t)(d0 + l) * ntargets + r;
        pot[row] += a[0];
        if (LEVEL >= 1 && level_out >= 1) {
          grad[row * 3 + 0] += a[1];
          grad[row * 3 + 1] += a[2];
          grad[row * 3 + 2] += a[3];
        }
        if (LEVEL >= 2 && level_out >= 2) {
          double* h = hess + row * 9;
          h[0] += a[4]; h[4] += a[5]; h[8] += a[6];
          h[1] += a[7]; h[3] += a[7];
          h[2] += a[8]; h[6] += a[8];
          h[5] += a[9]; h[7] += a[9];
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
// host dispatch

namespace {

constexpr int kBT = 64;   // 64-thread blocks x 2-4 targets/thread (tools/far_sweep.cu)
constexpr int kTS = 128;

struct ChunkSpec {
  int ndc, d0;
  bool hc, hd;
};

template <int NDC, bool HC, bool HD>
int launch_pack(const double* src, int64_t ns, int64_t ns_pad, const double* charges,
                const double* dipoles, int d0, uint32_t cmask, uint32_t dmask, double* out,
                cudaStream_t st) {
  const int64_t blocks = ceil_div(ns_pad, 256);
  pack_sources_kernel<NDC, HC, HD><<<(unsigned)blocks, 256, 0, st>>>(
      src, ns, ns_pad, charges, dipoles, ns, d0, cmask, dmask, out);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// the generic pair as an opfar functor: the direct sum reuses the stream-K
// sweep (one persistent wave, register-prefetched source tiles) of the
// operator far field
template <int NDC, bool HC, bool HD, int LEVEL>
struct GenericPairF {
  static constexpr int S = SrcLayout<NDC, HC, HD>::stride;
  static constexpr int NOUT = NDC * ncomp(LEVEL);
  static constexpr bool TN = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    pair_generic<NDC, HC, HD, LEVEL>(t.x, t.y, t.z, s, a);
  }
};

// stream-K partials -> reference layout (pot, grad, full hess), fixed order
__global__ void p2p_sk_finalize_kernel(const double* __restrict__ part, SkLayout L, int64_t nt,
                                       int ndc, int nc, int d0, int level, double* __restrict__ pot,
                                       double* __restrict__ grad, double* __restrict__ hess,
                                       int accumulate) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)ndc * nt) return;
  const int l = (int)(idx / nt);
  const int64_t i = idx - (int64_t)l * nt;
  const int na = ndc * nc;
  double v[10];
  for (int c = 0; c < nc; ++c) v[c] = sk_sum(part, L, na, l * nc + c, i);
  const int64_t row = (int64_t)(d0 + l) * nt + i;
  if (accumulate) pot[row] += v[0]; else pot[row] = v[0];
  if (level >= 1) {
    double* g = grad + row * 3;
    for (int k = 0; k < 3; ++k) { if (accumulate) g[k] += v[1 + k]; else g[k] = v[1 + k]; }
  }
  if (level >= 2) {
    const double hv[9] = {v[4], v[7], v[8], v[7], v[5], v[9], v[8], v[9], v[6]};
    double* h = hess + row * 9;
    for (int k = 0; k < 9; ++k) { if (accumulate) h[k] += hv[k]; else h[k] = hv[k]; }
  }
}

template <int NDC, bool HC, bool HD, int LEVEL>
int run_direct_chunk(const double* tgt, int64_t nt, const double* src, int64_t ns,
                     const double* charges, const double* dipoles, int d0, uint32_t cmask,
                     uint32_t dmask, int level_out, double* pot, double* grad, double* hess,
                     int accumulate, cudaStream_t st) {
  using F = GenericPairF<NDC, HC, HD, LEVEL>;
  constexpr int NA = F::NOUT;
  constexpr int NC = ncomp(LEVEL);
  constexpr int TPT = NA <= 4 ? 4 : (NA <= 12 ? 2 : 1);
  constexpr int TS = F::S <= 4 ? 64 : 128;  // tools/far_sweep.cu shapes
  constexpr int BT = 64;
  const int64_t ns_pad = ceil_div(ns, kTS) * kTS;  // kTS = 128 is a multiple of TS
  Scratch pack;
  LB_TRY(pack.alloc(sizeof(double) * ns_pad * F::S, st));
  LB_TRY((launch_pack<NDC, HC, HD>(src, ns, ns_pad, charges, dipoles, d0, cmask, dmask,
                                   pack.as<double>(), st)));
  auto kern = opfar_kernel<F, TPT, BT, TS>;
  static int per_sm = -1;
  if (per_sm < 0) {
    int b = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kern, BT, 0);
    per_sm = std::max(b, 1);
  }
  const SkLayout L = make_sk_layout(nt, ns_pad, BT * TPT, TS, (int64_t)sm_count() * per_sm);
  Scratch part;
  LB_TRY(part.alloc(sizeof(double) * L.tiles * L.kmax * NA * L.tt, st));
  kern<<<(unsigned)L.G, BT, 0, st>>>(tgt, nullptr, nt, pack.as<double>(), L, part.as<double>(), nullptr);
  LB_CHECK_LAUNCH();
  const int64_t nfin = (int64_t)NDC * nt;
  p2p_sk_finalize_kernel<<<(unsigned)ceil_div(nfin, 256), 256, 0, st>>>(
      part.as<double>(), L, nt, NDC, NC, d0, level_out, pot, grad, hess, accumulate);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

template <int NDC, bool HC, bool HD, int LEVEL>
int run_grouped_chunk(const double* t_xyz, const int64_t* t_out, const int64_t* t_off,
                      int64_t ngroups, const double* s_xyz, const double* s_c,
                      const double* s_v, const int64_t* s_off, int64_t nsf, int d0,
                      uint32_t cmask, uint32_t dmask, int level_out, int64_t ntargets,
                      double* pot, double* grad, double* hess, cudaStream_t st) {
  using L = SrcLayout<NDC, HC, HD>;
  Scratch pack;
  LB_TRY(pack.alloc(sizeof(double) * std::max<int64_t>(nsf, 1) * L::stride, st));
  if (nsf > 0)
    LB_TRY((launch_pack<NDC, HC, HD>(s_xyz, nsf, nsf, s_c, s_v, d0, cmask, dmask,
                                     pack.as<double>(), st)));
  if (ngroups > 0) {
    p2p_grouped_kernel<NDC, HC, HD, LEVEL, kBT, 64><<<(unsigned)ngroups, kBT, 0, st>>>(
        t_xyz, t_out, t_off, pack.as<double>(), s_off, ntargets, d0, level_out, pot, grad, hess);
    LB_CHECK_LAUNCH();
  }
  return LB_OK;
}

// runtime -> template dispatch over (ndc, hc, hd, level)
template <template <int, bool, bool, int> class F, class... A>
int dispatch(const ChunkSpec& c, int level, A... a) {
#define LB_CASE(N, C, D, LV) \
  if (c.ndc == N && c.hc == C && c.hd == D && level == LV) return F<N, C, D, LV>::run(a...);
#define LB_LV(N, C, D) LB_CASE(N, C, D, 0) LB_CASE(N, C, D, 1) LB_CASE(N, C, D, 2)
#define LB_CD(N) LB_LV(N, true, false) LB_LV(N, false, true) LB_LV(N, true, true)
  LB_CD(1) LB_CD(2) LB_CD(3) LB_CD(4)
#undef LB_CD
#undef LB_LV
#undef LB_CASE
  return fail(LB_ERR_ARG, "p2p: unsupported density chunk");
}

template <int N, bool C, bool D, int LV>
struct DirectF {
  template <class... A>
  static int run(A... a) { return run_direct_chunk<N, C, D, LV>(a...); }
};
template <int N, bool C, bool D, int LV>
struct GroupedF {
  template <class... A>
  static int run(A... a) { return run_grouped_chunk<N, C, D, LV>(a...); }
};

// split nd densities into chunks of <= 4 sharing the geometry work
std::vector<ChunkSpec> make_chunks(int nd, uint32_t cmask, uint32_t dmask) {
  std::vector<ChunkSpec> out;
  for (int d0 = 0; d0 < nd; d0 += 4) {
    ChunkSpec c;
    c.d0 = d0;
    c.ndc = std::min(4, nd - d0);
    uint32_t bits = ((c.ndc == 32) ? 0xffffffffu : ((1u << c.ndc) - 1u)) << d0;
    c.hc = (cmask & bits) != 0;
    c.hd = (dmask & bits) != 0;
    out.push_back(c);
  }
  return out;
}

}  // namespace
}  // namespace lb

extern "C" {

int lb_p2p(const double* tgt, int64_t nt, const double* src, int64_t ns, const double* charges,
           const double* dipoles, int nd, uint32_t cmask, uint32_t dmask, int level, double* pot,
           double* grad, double* hess, int accumulate, void* stream) {
  using namespace lb;
  if (nd <= 0 || nd > 32) return fail(LB_ERR_SHAPE, "lb_p2p: nd must be in [1, 32]");
  if (level < 0 || level > 2) return fail(LB_ERR_ARG, "lb_p2p: level must be 0, 1 or 2");
  if (nt < 0 || ns < 0) return fail(LB_ERR_SHAPE, "lb_p2p: negative sizes");
  if (nt == 0) return LB_OK;
  if (!pot || (level >= 1 && !grad) || (level >= 2 && !hess))
    return fail(LB_ERR_ARG, "lb_p2p: missing output buffer for the requested level");
  if ((cmask && !charges) || (dmask && !dipoles))
    return fail(LB_ERR_ARG, "lb_p2p: active mask without a density array");
  if (nt == 0) return LB_OK;
  cudaStream_t st = as_stream(stream);
  uint32_t valid = nd == 32 ? 0xffffffffu : ((1u << nd) - 1u);
  cmask &= valid;
  dmask &= valid;
  if (ns == 0 || (cmask | dmask) == 0) {
    if (!accumulate) {
      LB_CUDA(cudaMemsetAsync(pot, 0, sizeof(double) * nd * nt, st));
      if (level >= 1) LB_CUDA(cudaMemsetAsync(grad, 0, sizeof(double) * nd * nt * 3, st));
      if (level >= 2) LB_CUDA(cudaMemsetAsync(hess, 0, sizeof(double) * nd * nt * 9, st));
    }
    return LB_OK;
  }
  for (const ChunkSpec& c : make_chunks(nd, cmask, dmask)) {
    if (!c.hc && !c.hd) {
      if (!accumulate) {
        LB_CUDA(cudaMemsetAsync(pot + (int64_t)c.d0 * nt, 0, sizeof(double) * c.ndc * nt, st));
        if (level >= 1)
          LB_CUDA(cudaMemsetAsync(grad + (int64_t)c.d0 * nt * 3, 0, sizeof(double) * c.ndc * nt * 3, st));
        if (level >= 2)
          LB_CUDA(cudaMemsetAsync(hess + (int64_t)c.d0 * nt * 9, 0, sizeof(double) * c.ndc * nt * 9, st));
      }
      continue;
    }
    LB_TRY((dispatch<DirectF>(c, level, tgt, nt, src, ns, charges, dipoles, c.d0, cmask, dmask,
                              level, pot, grad, hess, accumulate, st)));
  }
  return LB_OK;
}

int lb_p2p_grouped(const double* t_xyz, const int64_t* t_out, const int64_t* t_off,
                   int64_t ngroups, int64_t ntf, const double* s_xyz, const double* s_c,
                   const double* s_v, const int64_t* s_off, int64_t nsf, int nd, uint32_t cmask,
                   uint32_t dmask, int level, int64_t ntargets, double* pot, double* grad,
                   double* hess, void* stream) {
  using namespace lb;
  (void)ntf;
  if (nd <= 0 || nd > 32) return fail(LB_ERR_SHAPE, "lb_p2p_grouped: nd must be in [1, 32]");
  if (level < 0 || level > 2) return fail(LB_ERR_ARG, "lb_p2p_grouped: level must be 0, 1 or 2");
  if (!pot || (level >= 1 && !grad) || (level >= 2 && !hess))
    return fail(LB_ERR_ARG, "lb_p2p_grouped: missing output buffer for the requested level");
  if ((cmask && !s_c) || (dmask && !s_v))
    return fail(LB_ERR_ARG, "lb_p2p_grouped: active mask without a density array");
  if (ngroups <= 0 || nsf <= 0) return LB_OK;
  cudaStream_t st = as_stream(stream);
  uint32_t valid = nd == 32 ? 0xffffffffu : ((1u << nd) - 1u);
  cmask &= valid;
  dmask &= valid;
  for (const ChunkSpec& c : make_chunks(nd, cmask, dmask)) {
    if (!c.hc && !c.hd) continue;
    LB_TRY((dispatch<GroupedF>(c, level, t_xyz, t_out, t_off, ngroups, s_xyz, s_c, s_v, s_off,
                               nsf, c.d0, cmask, dmask, level, ntargets, pot, grad, hess, st)));
  }
  return LB_OK;
}

}  // extern "C"
