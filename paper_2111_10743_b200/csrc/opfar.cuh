// Far-field pair functors of the operator apply and the tiled all-pairs
// kernel that runs them (shared by opset.cu and the tuning harness).
#pragma once

#include <algorithm>
#include <type_traits>

#include "lb_common.cuh"

namespace lb {

constexpr double kInv4Pi = 0.079577471545947667884441881686257181;  // 1/(4 pi)

struct Tgt {
  double x, y, z, nx, ny, nz;
  double n3x, n3y, n3z, h;  // n/3 and -2H/3 (FarA3c only; dead elsewhere)
};

// Functors accumulate NACC values per target (default NOUT) and may project
// them onto the NOUT written outputs once per tile (finish(), reading the
// target normal from global memory then instead of holding it in registers).
template <class F, class = void>
struct FarTraits {
  static constexpr int NACC = F::NOUT;
  static constexpr bool PROJ = false;
  static constexpr bool TC = false;
};
template <class F>
struct FarTraits<F, std::void_t<decltype(F::NACC)>> {
  static constexpr int NACC = F::NACC;
  static constexpr bool PROJ = true;
  static constexpr bool TC = F::TC;
};

// ---------------------------------------------------------------------------
// far-field pair functors.  r = t - s; every functor skips r == 0 through
// inv_sqrt_skip.  Output j of functor F accumulates into a[j].

#define LB_GEOM                                                     \
  const double r0 = t.x - s[0], r1 = t.y - s[1], r2 = t.z - s[2];   \
  const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));              \
  const double invr = inv_sqrt_skip(rr);

// S (pot only):  a0 += c/r                      record [x y z c]
struct FarS {
  static constexpr int S = 4, NOUT = 1;
  static constexpr bool TN = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    a[0] = fma(s[3], invr, a[0]);
  }
};

// A3 call 1 (operators.py:237): charge c, pot + n_t.grad.
//   a0 += c/r ; a1..3 += c r/r^3, projected once per tile: out1 = n_t.a1..3
//   (n_t.grad = -out1).  Accumulating the vector (3 FMA) instead of n_t.r per
//   pair (3 ops + 1 FMA) saves one FP64 op per pair and keeps the normal out
//   of the registers.                                          record [x y z c]
struct FarA3a {
  static constexpr int S = 4, NOUT = 2, NACC = 4;
  static constexpr bool TN = false, TC = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double ci = s[3] * invr;
    const double ci3 = ci * (invr * invr);
    a[0] += ci;
    a[1] = fma(ci3, r0, a[1]);
    a[2] = fma(ci3, r1, a[2]);
    a[3] = fma(ci3, r2, a[3]);
  }
  __device__ static void finish(const double* nrm, const double* a, double* o) {
    o[0] = a[0];
    o[1] = fma(nrm[2], a[3], fma(nrm[1], a[2], nrm[0] * a[1]));
  }
};

// S''+D' kernel times r^3, in the form of kernels.py:60-67:
//   3 (n_t.r)(dn.r)/r^2 - n_t.dn,   dn = n_t - n_s.
// dn is formed FIRST: for nearby nodes n_t - n_s is exact (Sterbenz), so
// n_t.dn = O(r^2) keeps its relative accuracy; the algebraically equal
// |n_t|^2 - n_t.n_s (or the reference's separate n.H.n + n.grad_dipole,
// operators.py:257-259) loses ~eps/r^2 of it.  The sum equals
// n_t.hess(charge).n_t + n_t.grad(dipole n_s).
#define LB_SPP_TERMS                                                       \
  const double dn0 = t.nx - s[3], dn1 = t.ny - s[4], dn2 = t.nz - s[5];    \
  const double rnt = fma(t.nz, r2, fma(t.ny, r1, t.nx * r0));              \
  const double rdn = fma(dn2, r2, fma(dn1, r1, dn0 * r0));                 \
  const double ndn = fma(t.nz, dn2, fma(t.ny, dn1, t.nx * dn0));           \
  const double kspp = fma(3.0 * rnt * rdn, invr * invr, -ndn);

// A3 call 2 (operators.py:247-259): charges c0 = w mu1, c1 = w mu2 and
// dipole c1 n_s.   record [x y z nx ny nz c0 c1]
//   a0 += c0 (n_t.r)/r^3   (sp_mu1 far = -a0)
//   a1 += c1 / r           (s_mu2 far)
//   a2 += c1 (n_t.r)/r^3   (sp_mu2 far = -a2)
//   a3 += c1 Kspp/r^3      (sppdp_mu2 far)
struct FarA3b {
  static constexpr int S = 8, NOUT = 4;
  static constexpr bool TN = true;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double invr3 = invr * (invr * invr);
    LB_SPP_TERMS
    const double g = rnt * invr3;
    a[0] = fma(s[6], g, a[0]);
    a[1] = fma(s[7], invr, a[1]);
    a[2] = fma(s[7], g, a[2]);
    a[3] = fma(s[7] * invr3, kspp, a[3]);
  }
};

// A3 call 2 fused with its glue (operators.py:247-263, eta aside): the far
// part of  sp_mu1 - sppdp_mu2 - 2H sp_mu2  as ONE accumulator
//   a0 += r^-3 [ (n_t.r)(c0 - 2H c1) + c1 Kspp ],  result_far = -a0 / 4pi
// with Kspp = 3 (n_t.r)(dn.r)/r^2 - n_t.dn.  The factor 3 is folded into the
// record (slot 7 holds 3 c1, written by the oversample) and the target
// (n_t/3, -2H/3), so  Kspp/3 = (n_t.r)(dn.r)/r^2 - (n_t/3).dn:
// 31 FP64 ops per pair (FarA3b: 34) and one output instead of four; S[mu2]
// for the W-average comes from eta = <Phi, mu2> (Phi = S^T w, precomputed).
//   record [x y z nx ny nz c0 3c1]
struct FarA3c {
  static constexpr int S = 8, NOUT = 1, NACC = 1;
  static constexpr bool TN = true, TC = true;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double invr2 = invr * invr;
    const double invr3 = invr * invr2;
    const double dn0 = t.nx - s[3], dn1 = t.ny - s[4], dn2 = t.nz - s[5];
    const double rnt = fma(t.nz, r2, fma(t.ny, r1, t.nx * r0));
    const double rdn = fma(dn2, r2, fma(dn1, r1, dn0 * r0));
    const double ndn3 = fma(t.n3z, dn2, fma(t.n3y, dn1, t.n3x * dn0));
    const double c0p = fma(t.h, s[7], s[6]);              // c0 - 2H c1
    const double k3 = fma(rnt * rdn, invr2, -ndn3);       // Kspp / 3
    const double inner = fma(rnt, c0p, s[7] * k3);
    a[0] = fma(invr3, inner, a[0]);
  }
  __device__ static void finish(const double*, const double* a, double* o) { o[0] = a[0]; }
};

// A2 call 1 (operators.py:200-212): charge c and dipole c n_s (c = w tau).
//   a0 += c/r ; a1 += c (n_s.r)/r^3 (D) ; a2 += c (n_t.r)/r^3 ; a3 += c Kspp/r^3
//   record [x y z nx ny nz c 0]
struct FarA2a {
  static constexpr int S = 8, NOUT = 4;
  static constexpr bool TN = true;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double c = s[6];
    const double ci = c * invr;
    const double ci3 = ci * (invr * invr);
    LB_SPP_TERMS
    const double rns = rnt - rdn;  // n_s.r
    a[0] += ci;
    a[1] = fma(ci3, rns, a[1]);
    a[2] = fma(ci3, rnt, a[2]);
    a[3] = fma(ci3, kspp, a[3]);
  }
};

// A2 call 2 (operators.py:216-223): dipole c0 n_s (c0 = w mu1), charge c1 = w mu2
//   a0 += c0 (n_s.r)/r^3 ; a1 += c1/r      record [x y z nx ny nz c0 c1]
struct FarA2b {
  static constexpr int S = 8, NOUT = 2;
  static constexpr bool TN = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double rns = fma(s[5], r2, fma(s[4], r1, s[3] * r0));
    a[0] = fma(s[6] * rns, invr * (invr * invr), a[0]);
    a[1] = fma(s[7], invr, a[1]);
  }
};

// D alone (apply_layer DOUBLE_LAYER, operators.py:144-147): record [.. c0 ..]
struct FarD {
  static constexpr int S = 8, NOUT = 1;
  static constexpr bool TN = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double rns = fma(s[5], r2, fma(s[4], r1, s[3] * r0));
    a[0] = fma(s[6] * rns, invr * (invr * invr), a[0]);
  }
};

// A1 call 1 (operators.py:167-171): charge c, pot + full gradient
//   a0 += c/r ; a1..3 += c r/r^3  (grad = -a1..3)        record [x y z c]
struct FarA1a {
  static constexpr int S = 4, NOUT = 4;
  static constexpr bool TN = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double ci = s[3] * invr;
    const double ci3 = ci * (invr * invr);
    a[0] += ci;
    a[1] = fma(ci3, r0, a[1]);
    a[2] = fma(ci3, r1, a[2]);
    a[3] = fma(ci3, r2, a[3]);
  }
};

// A1 call 2 (operators.py:181-185): three charges c_l = w mu_l, only the
// divergence sum_l d_l u_l is consumed:  a0 += (c . r)/r^3 (div far = -a0)
//   record [x y z c0 c1 c2]
struct FarA1b {
  static constexpr int S = 6, NOUT = 1;
  static constexpr bool TN = false;
  __device__ static void pair(const Tgt& t, const double* s, double* a) {
    LB_GEOM
    const double cr = fma(s[5], r2, fma(s[4], r1, s[3] * r0));
    a[0] = fma(cr, invr * (invr * invr), a[0]);
  }
};

#undef LB_GEOM

// ---------------------------------------------------------------------------
// Stream-K all-pairs sweep.  The sweep is U = tiles x C work units (one
// BT*TPT-target tile against one TS-source tile); a persistent grid of G CTAs
// (one full wave) takes contiguous unit ranges in tile-major order, so every
// CTA does the same amount of fp64 work (no wave quantisation, no tail) and
// accumulates a run of source tiles for one target tile in registers before
// writing ONE partial per (tile, CTA).  Tile t's partials come from CTAs
// bfirst(t)..blast(t) and are stored at slot k = b - bfirst(t); the consumer
// sums them in slot order (deterministic).

struct SkLayout {
  int64_t tiles, C, G, U, kmax;
  int tt;  // targets per tile
  __host__ __device__ int64_t owner(int64_t x) const { return ((x + 1) * G + U - 1) / U - 1; }
  __host__ __device__ int64_t bfirst(int64_t t) const { return owner(t * C); }
  __host__ __device__ int64_t blast(int64_t t) const { return owner(t * C + C - 1); }
  // index of partial (tile t, slot k, output o, local target lt)
  __host__ __device__ int64_t idx(int64_t t, int64_t k, int o, int nout, int lt) const {
    return ((t * kmax + k) * nout + o) * (int64_t)tt + lt;
  }
};

inline SkLayout make_sk_layout(int64_t n, int64_t ns_pad, int tt, int ts, int64_t slots) {
  SkLayout L;
  L.tt = tt;
  L.tiles = (n + tt - 1) / tt;
  L.C = ns_pad / ts;
  L.U = L.tiles * L.C;
  L.G = std::max<int64_t>(1, std::min<int64_t>(slots, L.U));
  L.kmax = std::min<int64_t>(L.C, (L.G + L.tiles - 1) / L.tiles + 1);
  return L;
}

// sum of the partials of output o for target i (consumer side)
__device__ __forceinline__ double sk_sum(const double* __restrict__ part, const SkLayout& L, int nout,
                                         int o, int64_t i) {
  const int64_t t = i / L.tt;
  const int lt = (int)(i - t * L.tt);
  const int64_t ns = L.blast(t) - L.bfirst(t) + 1;
  double v = 0.0;
  for (int64_t k = 0; k < ns; ++k) v += part[L.idx(t, k, o, nout, lt)];
  return v;
}

template <class F, int TPT, int BT, int TS, bool PF = true, int UR = 4, int MINB = 1>
__global__ void __launch_bounds__(BT, MINB) opfar_kernel(const double* __restrict__ nodes,
                                                   const double* __restrict__ normals, int64_t n,
                                                   const double* __restrict__ pack, SkLayout L,
                                                   double* __restrict__ part,
                                                   const double* __restrict__ curv = nullptr) {
  using Tr = FarTraits<F>;
  constexpr int S = F::S;
  constexpr int NO = F::NOUT;
  constexpr int NA = Tr::NACC;
  __shared__ __align__(16) double sh[TS * S];
  const int64_t b = blockIdx.x;
  int64_t u = b * L.U / L.G;
  const int64_t u_end = (b + 1) * L.U / L.G;
  while (u < u_end) {
    const int64_t t = u / L.C;
    const int64_t c0 = u - t * L.C;
    const int64_t c1 = min(L.C, c0 + (u_end - u));
    Tgt tg[TPT];
    double acc[TPT][NA];
#pragma unroll
    for (int j = 0; j < TPT; ++j) {
      const int64_t i = t * (BT * TPT) + (int64_t)j * BT + threadIdx.x;
      const bool in = i < n;
      tg[j].x = in ? nodes[3 * i] : 0.0;
      tg[j].y = in ? nodes[3 * i + 1] : 0.0;
      tg[j].z = in ? nodes[3 * i + 2] : 0.0;
      if (F::TN) {
        tg[j].nx = in ? normals[3 * i] : 0.0;
        tg[j].ny = in ? normals[3 * i + 1] : 0.0;
        tg[j].nz = in ? normals[3 * i + 2] : 0.0;
      } else {
        tg[j].nx = tg[j].ny = tg[j].nz = 0.0;
      }
      if (Tr::TC) {
        tg[j].n3x = tg[j].nx * (1.0 / 3.0);
        tg[j].n3y = tg[j].ny * (1.0 / 3.0);
        tg[j].n3z = tg[j].nz * (1.0 / 3.0);
        tg[j].h = in ? curv[i] * (-2.0 / 3.0) : 0.0;
      }
#pragma unroll
      for (int o = 0; o < NA; ++o) acc[j][o] = 0.0;
    }
    // the next source tile is prefetched into registers while the current
    // one is consumed from shared memory (hides the L2 latency behind fp64
    // work instead of stalling every CTA on the same barrier)
    constexpr int NPF = (TS * S / 2 + BT - 1) / BT;
    double2 pf[PF ? NPF : 1];
    if (PF) {
      const double2* g = reinterpret_cast<const double2*>(pack + c0 * TS * S);
#pragma unroll
      for (int q = 0; q < NPF; ++q) {
        const int k = q * BT + threadIdx.x;
        if (k < TS * S / 2) pf[q] = __ldg(g + k);
      }
    }
    for (int64_t c = c0; c < c1; ++c) {
      __syncthreads();
      double2* d = reinterpret_cast<double2*>(sh);
      if (PF) {
#pragma unroll
        for (int q = 0; q < NPF; ++q) {
          const int k = q * BT + threadIdx.x;
          if (k < TS * S / 2) d[k] = pf[q];
        }
      } else {
        const double2* g = reinterpret_cast<const double2*>(pack + c * TS * S);
#pragma unroll 4
        for (int k = threadIdx.x; k < TS * S / 2; k += BT) d[k] = __ldg(g + k);
      }
      __syncthreads();
      if (PF && c + 1 < c1) {
        const double2* g = reinterpret_cast<const double2*>(pack + (c + 1) * TS * S);
#pragma unroll
        for (int q = 0; q < NPF; ++q) {
          const int k = q * BT + threadIdx.x;
          if (k < TS * S / 2) pf[q] = __ldg(g + k);
        }
      }
#pragma unroll UR
      for (int k = 0; k < TS; ++k) {
#pragma unroll
        for (int j = 0; j < TPT; ++j) F::pair(tg[j], sh + k * S, acc[j]);
      }
    }
    const int64_t k = b - L.bfirst(t);
#pragma unroll
    for (int j = 0; j < TPT; ++j) {
      double out[NO];
      if constexpr (Tr::PROJ) {
        const int64_t i = min(n - 1, t * (BT * TPT) + (int64_t)j * BT + threadIdx.x);
        F::finish(normals + 3 * i, acc[j], out);
      } else {
#pragma unroll
        for (int o = 0; o < NO; ++o) out[o] = acc[j][o];
      }
#pragma unroll
      for (int o = 0; o < NO; ++o) part[L.idx(t, k, o, NO, j * BT + threadIdx.x)] = out[o];
    }
    u += c1 - c0;
  }
}

}  // namespace lb
