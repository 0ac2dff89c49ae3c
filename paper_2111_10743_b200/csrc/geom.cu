// Surface geometry from per-patch chart expansions: the device half of
// build_from_coefficients (surface.py:176-307), which the lbmesh reader
// (meshio.py:35-50) ends in.  One CTA per patch; every stage is a small
// (points x nb) x (nb x 3) product against a reference-element table that
// all CTAs share through L1/L2, so the kernel is latency-bound setup work
// (microseconds for config 2, ~1 ms at config 4's 26,732 patches), not a
// roofline kernel.
#include <cstdint>

#include "lb_common.cuh"

namespace lb {
namespace {

constexpr int kGeomThreads = 128;

__device__ __forceinline__ void smem_max(unsigned long long* a, double v) {
  atomicMax(a, (unsigned long long)__double_as_longlong(v));  // v >= 0
}
__device__ __forceinline__ void smem_min(unsigned long long* a, double v) {
  atomicMin(a, (unsigned long long)__double_as_longlong(v));  // v >= 0
}

// rows [r0, r1) of `tab` (rows x nb) applied to the (nb, 3) expansion c.
__device__ __forceinline__ void eval3(const double* __restrict__ row, const double* c, int nb,
                                      double& x, double& y, double& z) {
  x = y = z = 0.0;
  for (int j = 0; j < nb; ++j) {
    const double p = __ldg(row + j);
    x = fma(p, c[3 * j], x);
    y = fma(p, c[3 * j + 1], y);
    z = fma(p, c[3 * j + 2], z);
  }
}

__device__ __forceinline__ double cross_norm(double ax, double ay, double az, double bx, double by,
                                             double bz, double& cx, double& cy, double& cz) {
  cx = ay * bz - az * by;
  cy = az * bx - ax * bz;
  cz = ax * by - ay * bx;
  return sqrt(cx * cx + cy * cy + cz * cz);
}

__global__ void geom_stats_init(double* stats) {
  stats[0] = 0.0;
  stats[1] = 0.0;
  stats[2] = __longlong_as_double(0x7ff0000000000000LL);
  stats[3] = __longlong_as_double(0x7ff0000000000000LL);
  stats[4] = 0.0;
  stats[5] = 0.0;
}

__global__ void __launch_bounds__(kGeomThreads) geom_kernel(const lb_geom_desc d) {
  extern __shared__ double sm[];
  const int nb = d.nb, nq = d.nq, no = d.no, nloc = d.no / 4;
  const int64_t p = blockIdx.x;
  double* cx = sm;                  // (nb, 3) x 3 expansions
  double* cu = cx + 3 * nb;
  double* cv = cu + 3 * nb;
  double* X = cv + 3 * nb;          // node values (nb, 3)
  double* Xu = X + 3 * nb;
  double* Xv = Xu + 3 * nb;
  double* jw = Xv + 3 * nb;         // jr * rule_wts (nq), then 4 x nq child weights
  __shared__ unsigned long long red[4];
  __shared__ double sums[2];
  const int t = threadIdx.x;
  if (t < 4) red[t] = (t < 2) ? 0ull : 0x7ff0000000000000ull;
  if (t < 2) sums[t] = 0.0;
  for (int i = t; i < 3 * nb; i += blockDim.x) {
    cx[i] = d.coeffs_x[p * 3 * nb + i];
    cu[i] = d.coeffs_dxdu[p * 3 * nb + i];
    cv[i] = d.coeffs_dxdv[p * 3 * nb + i];
  }
  __syncthreads();

  // coefficient norms for the tail check (surface.py:205-207): the top total
  // degree is the last `order` columns of the degree-major basis
  {
    double all = 0.0, top = 0.0;
    for (int i = t; i < 3 * nb; i += blockDim.x) {
      const double s = cx[i] * cx[i];
      all += s;
      if (i / 3 >= nb - d.order) top += s;
    }
    atomicAdd(&sums[0], top);
    atomicAdd(&sums[1], all);
  }

  // nodes and stored tangents (surface.py:193-195)
  const int64_t n0 = p * nb;
  for (int i = t; i < nb; i += blockDim.x) {
    const double* row = d.vand + (int64_t)i * nb;
    double a, b, c;
    eval3(row, cx, nb, a, b, c);
    X[3 * i] = a; X[3 * i + 1] = b; X[3 * i + 2] = c;
    d.nodes[3 * (n0 + i)] = a; d.nodes[3 * (n0 + i) + 1] = b; d.nodes[3 * (n0 + i) + 2] = c;
    eval3(row, cu, nb, a, b, c);
    Xu[3 * i] = a; Xu[3 * i + 1] = b; Xu[3 * i + 2] = c;
    d.tangents_u[3 * (n0 + i)] = a; d.tangents_u[3 * (n0 + i) + 1] = b; d.tangents_u[3 * (n0 + i) + 2] = c;
    eval3(row, cv, nb, a, b, c);
    Xv[3 * i] = a; Xv[3 * i + 1] = b; Xv[3 * i + 2] = c;
    d.tangents_v[3 * (n0 + i)] = a; d.tangents_v[3 * (n0 + i) + 1] = b; d.tangents_v[3 * (n0 + i) + 2] = c;
  }
  __syncthreads();

  // per node: consistency, normal, metric, curvature (surface.py:201-248)
  for (int i = t; i < nb; i += blockDim.x) {
    const double* ru = d.dmat_u + (int64_t)i * nb;
    const double* rv = d.dmat_v + (int64_t)i * nb;
    double su[3] = {0, 0, 0}, sv[3] = {0, 0, 0};
    double uu[3] = {0, 0, 0}, uv1[3] = {0, 0, 0}, uv2[3] = {0, 0, 0}, vv[3] = {0, 0, 0};
    for (int j = 0; j < nb; ++j) {
      const double a = __ldg(ru + j), b = __ldg(rv + j);
#pragma unroll
      for (int c = 0; c < 3; ++c) {
        su[c] = fma(a, X[3 * j + c], su[c]);
        sv[c] = fma(b, X[3 * j + c], sv[c]);
        uu[c] = fma(a, Xu[3 * j + c], uu[c]);
        uv1[c] = fma(b, Xu[3 * j + c], uv1[c]);
        uv2[c] = fma(a, Xv[3 * j + c], uv2[c]);
        vv[c] = fma(b, Xv[3 * j + c], vv[c]);
      }
    }
    const double* xu = Xu + 3 * i;
    const double* xv = Xv + 3 * i;
    double mis = 0.0, mag = 0.0;
#pragma unroll
    for (int c = 0; c < 3; ++c) {
      mis = fmax(mis, fmax(fabs(su[c] - xu[c]), fabs(sv[c] - xv[c])));
      mag = fmax(mag, fmax(fabs(xu[c]), fabs(xv[c])));
    }
    double nx, ny, nz;
    const double jac = cross_norm(xu[0], xu[1], xu[2], xv[0], xv[1], xv[2], nx, ny, nz);
    nx /= jac; ny /= jac; nz /= jac;
    const double g11 = xu[0] * xu[0] + xu[1] * xu[1] + xu[2] * xu[2];
    const double g12 = xu[0] * xv[0] + xu[1] * xv[1] + xu[2] * xv[2];
    const double g22 = xv[0] * xv[0] + xv[1] * xv[1] + xv[2] * xv[2];
    const double det = g11 * g22 - g12 * g12;
    const double i00 = g22 / det, i01 = -g12 / det, i11 = g11 / det;
    const double b11 = nx * uu[0] + ny * uu[1] + nz * uu[2];
    const double b12 = nx * 0.5 * (uv1[0] + uv2[0]) + ny * 0.5 * (uv1[1] + uv2[1]) +
                       nz * 0.5 * (uv1[2] + uv2[2]);
    const double b22 = nx * vv[0] + ny * vv[1] + nz * vv[2];
    const int64_t g = n0 + i;
    d.normals[3 * g] = nx; d.normals[3 * g + 1] = ny; d.normals[3 * g + 2] = nz;
    d.metric[4 * g] = g11; d.metric[4 * g + 1] = g12; d.metric[4 * g + 2] = g12; d.metric[4 * g + 3] = g22;
    d.inv_metric[4 * g] = i00; d.inv_metric[4 * g + 1] = i01;
    d.inv_metric[4 * g + 2] = i01; d.inv_metric[4 * g + 3] = i11;
    d.sqrt_det_g[g] = jac;
    d.curvature[g] = -0.5 * (i00 * b11 + 2.0 * i01 * b12 + i11 * b22);
    smem_max(&red[0], mis);
    smem_max(&red[1], mag);
    smem_min(&red[2], jac);
  }

  // smooth node weights: |X_u x X_v| on the order-(p+1) rule, pulled back
  // through weight_interp (surface.py:250-255)
  for (int q = t; q < nq; q += blockDim.x) {
    const double* row = d.psi_rule + (int64_t)q * nb;
    double ax, ay, az, bx, by, bz, c0, c1, c2;
    eval3(row, cu, nb, ax, ay, az);
    eval3(row, cv, nb, bx, by, bz);
    jw[q] = cross_norm(ax, ay, az, bx, by, bz, c0, c1, c2) * __ldg(d.rule_wts + q);
  }
  // oversampled nodes and normals (surface.py:257-267)
  const int64_t o0 = p * no;
  for (int o = t; o < no; o += blockDim.x) {
    const double* row = d.psi_over + (int64_t)o * nb;
    double a, b, c, ax, ay, az, bx, by, bz;
    eval3(row, cx, nb, a, b, c);
    eval3(row, cu, nb, ax, ay, az);
    eval3(row, cv, nb, bx, by, bz);
    double nx, ny, nz;
    const double jac = cross_norm(ax, ay, az, bx, by, bz, nx, ny, nz);
    const int64_t g = o0 + o;
    d.over_nodes[3 * g] = a; d.over_nodes[3 * g + 1] = b; d.over_nodes[3 * g + 2] = c;
    d.over_normals[3 * g] = nx / jac; d.over_normals[3 * g + 1] = ny / jac;
    d.over_normals[3 * g + 2] = nz / jac;
    smem_min(&red[3], jac);
  }
  // the same rule on each child triangle, x 1/4 (surface.py:269-283)
  double* jc = jw + nq;
  for (int r = t; r < 4 * nq; r += blockDim.x) {
    const double* row = d.psi_child + (int64_t)r * nb;
    double ax, ay, az, bx, by, bz, c0, c1, c2;
    eval3(row, cu, nb, ax, ay, az);
    eval3(row, cv, nb, bx, by, bz);
    jc[r] = cross_norm(ax, ay, az, bx, by, bz, c0, c1, c2) * __ldg(d.rule_wts + r % nq) * 0.25;
  }
  __syncthreads();
  for (int i = t; i < nb; i += blockDim.x) {
    double w = 0.0;
    for (int q = 0; q < nq; ++q) w = fma(__ldg(d.weight_interp + (int64_t)q * nb + i), jw[q], w);
    d.weights[n0 + i] = w;
  }
  for (int o = t; o < no; o += blockDim.x) {
    const int k = o / nloc, i = o % nloc;
    double w = 0.0;
    for (int q = 0; q < nq; ++q) w = fma(__ldg(d.w_interp_o + (int64_t)q * nloc + i), jc[k * nq + q], w);
    d.over_weights[o0 + o] = w;
  }
  if (t == 0) {
    atomicMax(reinterpret_cast<unsigned long long*>(d.stats + 0), red[0]);
    atomicMax(reinterpret_cast<unsigned long long*>(d.stats + 1), red[1]);
    atomicMin(reinterpret_cast<unsigned long long*>(d.stats + 2), red[2]);
    atomicMin(reinterpret_cast<unsigned long long*>(d.stats + 3), red[3]);
    atomicAdd(d.stats + 4, sums[0]);
    atomicAdd(d.stats + 5, sums[1]);
  }
}

}  // namespace
}  // namespace lb

extern "C" int lb_geom_build(const lb_geom_desc* d, void* stream) {
  using namespace lb;
  if (!d) return fail(LB_ERR_ARG, "lb_geom_build: null descriptor");
  if (d->order < 2 || d->order > 12 || d->nb != d->order * (d->order + 1) / 2)
    return fail(LB_ERR_SHAPE, "lb_geom_build: coefficient arrays do not match the stated order");
  if (d->nq < 1 || d->no < 4 || d->no % 4 != 0 || d->npatches < 0)
    return fail(LB_ERR_SHAPE, "lb_geom_build: bad table sizes");
  const void* need[] = {d->coeffs_x, d->coeffs_dxdu, d->coeffs_dxdv, d->vand, d->dmat_u,
                        d->dmat_v, d->psi_rule, d->rule_wts, d->weight_interp, d->psi_over,
                        d->psi_child, d->w_interp_o, d->nodes, d->tangents_u, d->tangents_v,
                        d->normals, d->metric, d->inv_metric, d->sqrt_det_g, d->curvature,
                        d->weights, d->over_nodes, d->over_normals, d->over_weights, d->stats};
  for (const void* q : need)
    if (!q) return fail(LB_ERR_ARG, "lb_geom_build: null pointer");
  cudaStream_t st = as_stream(stream);
  geom_stats_init<<<1, 1, 0, st>>>(d->stats);
  LB_CHECK_LAUNCH();
  if (d->npatches == 0) return LB_OK;
  const size_t smem = sizeof(double) * (18 * (size_t)d->nb + 5 * (size_t)d->nq);
  if (smem > 48 * 1024)
    LB_CUDA(cudaFuncSetAttribute(geom_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  geom_kernel<<<(unsigned)d->npatches, kGeomThreads, smem, st>>>(*d);
  LB_CHECK_LAUNCH();
  return LB_OK;
}
