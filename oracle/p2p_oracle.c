/*
 * TEST INFRASTRUCTURE ONLY — the CPU oracle for the hot path.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
 * may load this library; the product (paper_2111_10743_b200) never does.
 *
 * Plain-C restatement of the reference's pairwise kernels:
 *   - oracle_p2p: the per-pair formulas of grouped_direct
 *     (/root/reference/pkg/src/lapbel/_pointsum.py:33-89) over ALL
 *     target/source pairs, i.e. evaluate_direct (fmm.py:215-222): r == 0
 *     pairs skipped (fmm.py:136-141), charges and dipoles per density,
 *     level 0/1/2 = pot / +grad / +hess, Hessian upper triangle accumulated
 *     then mirrored (_pointsum.py:105-108).  OpenMP over targets mirrors the
 *     numba prange over target groups (_pointsum.py:30).
 *   - oracle_p2p_grouped: grouped_direct itself (_pointsum.py:19-89).
 *   - oracle_csr_matvec: y = A x for a scipy CSR matrix, the
 *     `self.corr(kind) @ tau` products of operators.py:155,239-259.
 * Strict IEEE arithmetic (compiled without -ffast-math), 1/sqrt(r2) exactly
 * as the reference writes it.
 */
#include <math.h>
#include <stdint.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

static void pair_all(double tx, double ty, double tz, const double* s_xyz,
                     int64_t si, const double* s_c, const double* s_v,
                     int64_t s_stride, int nd, uint32_t cmask, uint32_t dmask,
                     int level, double* acc /* nd*10 */) {
  const double r0 = tx - s_xyz[3 * si + 0];
  const double r1 = ty - s_xyz[3 * si + 1];
  const double r2 = tz - s_xyz[3 * si + 2];
  const double rr = r0 * r0 + r1 * r1 + r2 * r2;
  if (rr == 0.0) return;
  const double invr = 1.0 / sqrt(rr);
  const double invr3 = invr / rr;
  const double invr5 = invr3 / rr;
  for (int l = 0; l < nd; ++l) {
    double* a = acc + 10 * l;
    if ((cmask >> l) & 1u) {
      const double c = s_c[(int64_t)l * s_stride + si];
      if (c != 0.0) {
        a[0] += c * invr;
        if (level >= 1) {
          a[1] -= c * r0 * invr3;
          a[2] -= c * r1 * invr3;
          a[3] -= c * r2 * invr3;
        }
        if (level >= 2) {
          const double ci5 = 3.0 * c * invr5;
          a[4] += ci5 * r0 * r0 - c * invr3; /* xx */
          a[5] += ci5 * r1 * r1 - c * invr3; /* yy */
          a[6] += ci5 * r2 * r2 - c * invr3; /* zz */
          a[7] += ci5 * r0 * r1;             /* xy */
          a[8] += ci5 * r0 * r2;             /* xz */
          a[9] += ci5 * r1 * r2;             /* yz */
        }
      }
    }
    if ((dmask >> l) & 1u) {
      const double* v = s_v + ((int64_t)l * s_stride + si) * 3;
      const double v0 = v[0], v1 = v[1], v2 = v[2];
      const double vr = v0 * r0 + v1 * r1 + v2 * r2;
      a[0] += vr * invr3;
      if (level >= 1) {
        const double vr3 = 3.0 * vr * invr5;
        a[1] += v0 * invr3 - vr3 * r0;
        a[2] += v1 * invr3 - vr3 * r1;
        a[3] += v2 * invr3 - vr3 * r2;
      }
      if (level >= 2) {
        const double invr7 = invr5 / rr;
        const double w15 = 15.0 * vr * invr7;
        const double i5 = 3.0 * invr5;
        a[4] += w15 * r0 * r0 - i5 * (2.0 * v0 * r0 + vr);
        a[5] += w15 * r1 * r1 - i5 * (2.0 * v1 * r1 + vr);
        a[6] += w15 * r2 * r2 - i5 * (2.0 * v2 * r2 + vr);
        a[7] += w15 * r0 * r1 - i5 * (v0 * r1 + v1 * r0);
        a[8] += w15 * r0 * r2 - i5 * (v0 * r2 + v2 * r0);
        a[9] += w15 * r1 * r2 - i5 * (v1 * r2 + v2 * r1);
      }
    }
  }
}

static void store(const double* a, int nd, int64_t nt, int64_t row, int level,
                  double* pot, double* grad, double* hess, int accumulate) {
  for (int l = 0; l < nd; ++l) {
    const double* v = a + 10 * l;
    const int64_t r = (int64_t)l * nt + row;
    pot[r] = (accumulate ? pot[r] : 0.0) + v[0];
    if (level >= 1)
      for (int k = 0; k < 3; ++k)
        grad[3 * r + k] = (accumulate ? grad[3 * r + k] : 0.0) + v[1 + k];
    if (level >= 2) {
      const double h[9] = {v[4], v[7], v[8], v[7], v[5], v[9], v[8], v[9], v[6]};
      for (int k = 0; k < 9; ++k)
        hess[9 * r + k] = (accumulate ? hess[9 * r + k] : 0.0) + h[k];
    }
  }
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* all pairs; nd <= 32; outputs overwritten (or accumulated) */
int oracle_p2p(const double* tgt, int64_t nt, const double* src, int64_t ns,
               const double* charges, const double* dipoles, int nd,
               uint32_t cmask, uint32_t dmask, int level, double* pot,
               double* grad, double* hess, int accumulate, int nthreads) {
  if (nd <= 0 || nd > 32) return 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t i = 0; i < nt; ++i) {
    double acc[32 * 10];
    memset(acc, 0, sizeof(double) * 10 * nd);
    for (int64_t j = 0; j < ns; ++j)
      pair_all(tgt[3 * i], tgt[3 * i + 1], tgt[3 * i + 2], src, j, charges,
               dipoles, ns, nd, cmask, dmask, level, acc);
    store(acc, nd, nt, i, level, pot, grad, hess, accumulate);
  }
  return 0;
}

/* grouped_direct (_pointsum.py:19-89): outputs are ADDED into rows t_out */
int oracle_p2p_grouped(const double* t_xyz, const int64_t* t_out,
                       const int64_t* t_off, int64_t ngroups,
                       const double* s_xyz, const double* s_c,
                       const double* s_v, const int64_t* s_off, int64_t nsf,
                       int nd, uint32_t cmask, uint32_t dmask, int level,
                       int64_t ntargets, double* pot, double* grad,
                       double* hess, int nthreads) {
  if (nd <= 0 || nd > 32) return 1;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
  for (int64_t g = 0; g < ngroups; ++g) {
    for (int64_t ti = t_off[g]; ti < t_off[g + 1]; ++ti) {
      double acc[32 * 10];
      memset(acc, 0, sizeof(double) * 10 * nd);
      for (int64_t si = s_off[g]; si < s_off[g + 1]; ++si)
        pair_all(t_xyz[3 * ti], t_xyz[3 * ti + 1], t_xyz[3 * ti + 2], s_xyz,
                 si, s_c, s_v, nsf, nd, cmask, dmask, level, acc);
      store(acc, nd, ntargets, t_out[ti], level, pot, grad, hess, 1);
    }
  }
  return 0;
}

/* y[i] (+)= sum_k data[k] x[indices[k]], k in indptr[i]:indptr[i+1] */
int oracle_csr_matvec(const int64_t* indptr, const int32_t* indices,
                      const double* data, int64_t nrows, const double* x,
                      double* y, int accumulate, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
  for (int64_t i = 0; i < nrows; ++i) {
    double s = 0.0;
    for (int64_t k = indptr[i]; k < indptr[i + 1]; ++k) s += data[k] * x[indices[k]];
    y[i] = (accumulate ? y[i] : 0.0) + s;
  }
  return 0;
}

/* The S''+D' far kernel in the combined form of kernels.py:60-67 (no 1/4pi):
 *   out_i = sum_j c_j (3 (nx.r)((nx-ny).r)/r^2 - nx.(nx-ny)) / r^3,
 * r = x_i - y_j, r == 0 skipped.  Algebraically equal to the reference's
 * separate n.H(charge).n + n.grad(dipole c n_y) (operators.py:257-259) but
 * without its 1/r^5 cancellation. */
int oracle_spp_far(const double* x, const double* nx, int64_t nt,
                   const double* y, const double* ny, const double* c,
                   int64_t ns, double* out, int nthreads) {
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t i = 0; i < nt; ++i) {
    double acc = 0.0;
    const double n0 = nx[3 * i], n1 = nx[3 * i + 1], n2 = nx[3 * i + 2];
    for (int64_t j = 0; j < ns; ++j) {
      const double r0 = x[3 * i] - y[3 * j], r1 = x[3 * i + 1] - y[3 * j + 1],
                   r2 = x[3 * i + 2] - y[3 * j + 2];
      const double rr = r0 * r0 + r1 * r1 + r2 * r2;
      if (rr == 0.0) continue;
      const double d0 = n0 - ny[3 * j], d1 = n1 - ny[3 * j + 1], d2 = n2 - ny[3 * j + 2];
      const double rnx = r0 * n0 + r1 * n1 + r2 * n2;
      const double rdn = r0 * d0 + r1 * d1 + r2 * d2;
      const double ndn = n0 * d0 + n1 * d1 + n2 * d2;
      const double invr = 1.0 / sqrt(rr);
      acc += c[j] * (3.0 * rnx * rdn / rr - ndn) * (invr / rr);
    }
    out[i] = acc;
  }
  return 0;
}
