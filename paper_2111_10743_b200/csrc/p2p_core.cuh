// Pairwise interaction core shared by the direct, grouped and FMM kernels.
//
// Per pair (target t, source s, r = t - s, density l), the formulas of
// _pointsum.py:46-89 / fmm.py:152-184:
//   charge c : pot += c/r
//              grad -= c r / r^3
//              hess += c (3 r r^T / r^5 - I / r^3)
//   dipole v : pot += (v.r) / r^3
//              grad += v / r^3 - 3 (v.r) r / r^5
//              hess += 15 (v.r) r r^T / r^7 - 3 (v r^T + r v^T + (v.r) I) / r^5
// Accumulator layout per density: [pot | gx gy gz | hxx hyy hzz hxy hxz hyz].
#pragma once

#include "lb_common.cuh"

namespace lb {

__host__ __device__ constexpr int ncomp(int level) {
  return 1 + (level >= 1 ? 3 : 0) + (level >= 2 ? 6 : 0);
}

// packed source record: x y z, then per density [c] [vx vy vz], padded to an
// even number of doubles so records stay 16-byte aligned in shared memory
template <int NDC, bool HC, bool HD>
struct SrcLayout {
  static constexpr int per_d = (HC ? 1 : 0) + (HD ? 3 : 0);
  static constexpr int raw = 3 + NDC * per_d;
  static constexpr int stride = (raw + 1) & ~1;
};

template <int NDC, bool HC, bool HD, int LEVEL>
__device__ __forceinline__ void pair_generic(double tx, double ty, double tz,
                                             const double* __restrict__ rec, double* acc) {
  constexpr int NC = ncomp(LEVEL);
  const double r0 = tx - rec[0];
  const double r1 = ty - rec[1];
  const double r2 = tz - rec[2];
  const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
  const double invr = inv_sqrt_skip(rr);
  const double invr2 = invr * invr;
  const double invr3 = invr * invr2;
  double invr5 = 0.0, invr7 = 0.0;
  if (LEVEL >= 2 || (LEVEL >= 1 && HD)) invr5 = invr3 * invr2;
  if (LEVEL >= 2 && HD) invr7 = invr5 * invr2;
  int o = 3;
#pragma unroll
  for (int l = 0; l < NDC; ++l) {
    double* a = acc + l * NC;
    if (HC) {
      const double c = rec[o++];
      a[0] = fma(c, invr, a[0]);
      if (LEVEL >= 1) {
        const double cr3 = c * invr3;
        a[1] = fma(-cr3, r0, a[1]);
        a[2] = fma(-cr3, r1, a[2]);
        a[3] = fma(-cr3, r2, a[3]);
        if (LEVEL >= 2) {
          const double ci5 = 3.0 * c * invr5;
          a[4] += fma(ci5 * r0, r0, -cr3);
          a[5] += fma(ci5 * r1, r1, -cr3);
          a[6] += fma(ci5 * r2, r2, -cr3);
          a[7] = fma(ci5 * r0, r1, a[7]);
          a[8] = fma(ci5 * r0, r2, a[8]);
          a[9] = fma(ci5 * r1, r2, a[9]);
        }
      }
    }
    if (HD) {
      const double v0 = rec[o++];
      const double v1 = rec[o++];
      const double v2 = rec[o++];
      const double vr = fma(v2, r2, fma(v1, r1, v0 * r0));
      a[0] = fma(vr, invr3, a[0]);
      if (LEVEL >= 1) {
        const double vr3 = 3.0 * vr * invr5;
        a[1] += fma(v0, invr3, -vr3 * r0);
        a[2] += fma(v1, invr3, -vr3 * r1);
        a[3] += fma(v2, invr3, -vr3 * r2);
        if (LEVEL >= 2) {
          const double w15 = 15.0 * vr * invr7;
          const double i5 = 3.0 * invr5;
          a[4] += fma(w15 * r0, r0, -i5 * fma(2.0 * v0, r0, vr));
          a[5] += fma(w15 * r1, r1, -i5 * fma(2.0 * v1, r1, vr));
          a[6] += fma(w15 * r2, r2, -i5 * fma(2.0 * v2, r2, vr));
          a[7] += fma(w15 * r0, r1, -i5 * fma(v0, r1, v1 * r0));
          a[8] += fma(w15 * r0, r2, -i5 * fma(v0, r2, v2 * r0));
          a[9] += fma(w15 * r1, r2, -i5 * fma(v1, r2, v2 * r1));
        }
      }
    }
  }
}

}  // namespace lb
