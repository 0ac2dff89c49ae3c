// Near-correction build on the device: the near map
// (build_near_map, quadrature.py:76-104) and the locally corrected rows
// (compute_corrections, quadrature.py:663-701) for the non-principal-value
// kinds S, D, S', S''+D'.
//
// Near map: one thread per target tests every patch's bounding sphere
// (patch tiles staged in shared memory), count pass + fill pass, own patch
// first then ascending patch index like the reference's list build.
//
// Adaptive rows (_adaptive_pairs, quadrature.py:277-420, leaf evaluation of
// _leafeval.py:64-190): ONE CTA per (target, patch) pair, pulled from a
// global work counter (persistent grid; self pairs carry ~50x the work and
// come first).  The CTA walks the pair's subdivision tree depth-first with an
// item stack in global scratch; every refinement evaluates the 2 (Duffy) or 4
// (smooth) children of one item as one batch: rule points spread over the
// CTA (Koornwinder basis by recurrence in registers, chart geometry from the
// patch's coefficients in shared memory, all kernels), then the basis-weighted
// sums as small dot products out of shared memory.  The accept test, tolerance
// and geometric forcing are the reference's; only the order of floating-point
// additions differs (the reference runs numba fastmath).
//
// Assembly (quadrature.py:558, 593-610, 690-700): rows = acc @ vinv minus the
// oversampled smooth rule composed with over_interp, written straight into the
// values of the sorted CSR pattern.
#include <cstdint>
#include <cstring>

#include "lb_common.cuh"

namespace lb {
namespace {

constexpr double kFourPi = 4.0 * 3.141592653589793;  // kernels.py:16
constexpr int kQuadThreads = 256;
constexpr int kMaxDepth = 30;                          // quadrature.py:43
constexpr int kStackItems = 128;                       // >= 3 + 3 * kMaxDepth
constexpr int kMaxKinds = 7;

// ---------------------------------------------------------------------------
// near map

constexpr int kNearTile = 512;

template <bool FILL>
__global__ void near_kernel(const double* __restrict__ nodes, int64_t n, const double* __restrict__ centers,
                            const double* __restrict__ rad, int64_t npat, const int64_t* __restrict__ node_patch,
                            int32_t* __restrict__ counts, const int64_t* __restrict__ offsets,
                            int32_t* __restrict__ patches) {
  __shared__ double sc[kNearTile * 4];
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = t < n;
  double x0 = 0, x1 = 0, x2 = 0;
  int64_t own = -1;
  int64_t slot = 0;
  if (live) {
    x0 = nodes[3 * t];
    x1 = nodes[3 * t + 1];
    x2 = nodes[3 * t + 2];
    own = node_patch[t];
    if (FILL) {
      slot = offsets[t];
      patches[slot++] = (int32_t)own;
    }
  }
  int cnt = 1;
  for (int64_t p0 = 0; p0 < npat; p0 += kNearTile) {
    const int m = (int)(npat - p0 < kNearTile ? npat - p0 : kNearTile);
    __syncthreads();
    for (int i = threadIdx.x; i < m; i += blockDim.x) {
      sc[4 * i] = centers[3 * (p0 + i)];
      sc[4 * i + 1] = centers[3 * (p0 + i) + 1];
      sc[4 * i + 2] = centers[3 * (p0 + i) + 2];
      sc[4 * i + 3] = rad[p0 + i];
    }
    __syncthreads();
    if (!live) continue;
    for (int i = 0; i < m; ++i) {
      // cKDTree.query_ball_point: squared distance (no FMA) <= r*r
      const double d0 = __dsub_rn(x0, sc[4 * i]), d1 = __dsub_rn(x1, sc[4 * i + 1]),
                   d2 = __dsub_rn(x2, sc[4 * i + 2]);
      const double dd = __dadd_rn(__dadd_rn(__dmul_rn(d0, d0), __dmul_rn(d1, d1)), __dmul_rn(d2, d2));
      const double r = sc[4 * i + 3];
      if (dd <= __dmul_rn(r, r) && p0 + i != own) {
        if (FILL) patches[slot++] = (int32_t)(p0 + i);
        else ++cnt;
      }
    }
  }
  if (!FILL && live) counts[t] = cnt;
}

// ---------------------------------------------------------------------------
// adaptive quadrature

struct QuadArgs {
  int nb, nk, nqs, nqd;
  int codes[kMaxKinds];
  double eps;
  const double* coeffs;      // (npat, nb, 9) x | dx/du | dx/dv, basis in k-major order
  const double* nodes;       // (N, 3)
  const double* normals;     // (N, 3)
  const double* node_uv;     // (N, 2)
  const int64_t* node_patch; // (N)
  const int64_t* pair_tgt;   // (npairs)
  const int32_t* pair_pat;   // (npairs)
  int64_t npairs;
  const double* srule;       // (nqs, 3): u, v, w      smooth leaf rule (triangle_rule(p+2))
  const double* drule;       // (nqd, 3): a, b, w      Duffy leaf rule
  const double* norm;        // (nb) Koornwinder normalisation, k-major
  double* acc;               // (npairs, nk, nb) k-major basis integrals
  double* stack;             // (gridDim.x, kStackItems, item)
  unsigned long long* next;  // work counter
  int* status;               // [0]: 0 ok / 1 depth cap
  long long* bad_pair;
  unsigned long long* stats; // [0] refinement steps, [1] leaves evaluated (optional)
  int mode;                  // 0: basis-weight rows (_row_integrand), 1: PV integrals (_pv_integrand)
  const double* hcoeff;      // mode 1: (npat, nb) mean-curvature coefficients, k-major
};

__host__ __device__ __forceinline__ bool is_grad(int code) { return code >= LB_KIND_GRAD_S1 && code <= LB_KIND_GRAD_S3; }

__global__ void self_pairs_kernel(const int64_t* __restrict__ node_patch, int64_t n, int64_t* __restrict__ tgt,
                                  int32_t* __restrict__ pat) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    tgt[i] = i;
    pat[i] = (int32_t)node_patch[i];
  }
}

// Koornwinder basis at (u, v), k-major (_leafeval.py:25-61)
template <int ORDER>
__device__ __forceinline__ void koornwinder_km(double u, double v, const double* __restrict__ norm, double* psi) {
  const double vm = fmin(v, 1.0 - 1e-14);
  const double a = 2.0 * u / (1.0 - vm) - 1.0;
  const double b = 2.0 * v - 1.0;
  const double one_m_v = 1.0 - vm;
  double leg[ORDER];
  leg[0] = 1.0;
  if (ORDER > 1) leg[1] = a;
#pragma unroll
  for (int n = 2; n < ORDER; ++n) leg[n] = ((2 * n - 1) * a * leg[n - 1] - (n - 1) * leg[n - 2]) / n;
  int col = 0;
  double powv = 1.0;
#pragma unroll
  for (int k = 0; k < ORDER; ++k) {
    const double alpha = 2.0 * k + 1.0;
    const double lk = leg[k] * powv;
    double qm1 = 1.0, qm2 = 0.0;
#pragma unroll
    for (int l = 0; l < ORDER - k; ++l) {
      double q;
      if (l == 0) {
        q = 1.0;
      } else if (l == 1) {
        q = ((alpha + 2.0) * b + alpha) / 2.0;
      } else {
        const double c0 = 2.0 * l * (l + alpha) * (2 * l + alpha - 2);
        const double c1 = (2 * l + alpha - 1) * (2 * l + alpha) * (2 * l + alpha - 2);
        const double c2 = (2 * l + alpha - 1) * alpha * alpha;
        const double c3 = 2.0 * (l + alpha - 1) * (l - 1) * (2 * l + alpha);
        q = ((c1 * b + c2) * qm1 - c3 * qm2) / c0;
      }
      psi[col] = norm[col] * lk * q;
      ++col;
      qm2 = qm1;
      qm1 = q;
    }
    powv *= one_m_v;
  }
}

template <int ORDER>
struct QuadShape {
  static constexpr int NB = ORDER * (ORDER + 1) / 2;
  static constexpr int NQ = (ORDER + 2) * (ORDER + 2);  // >= Duffy (p+2)(p+1)
  static constexpr int LB = NB * NQ * 4 * 8 <= 80 * 1024 ? 4 : 2;  // leaves per batch
  static constexpr int ITEM = 10 + kMaxKinds * NB;                 // verts 6, duffy, depth, mind, diam, vals
};

// shared-memory layout of one CTA
template <int ORDER>
struct QuadSmem {
  using Sh = QuadShape<ORDER>;
  double coeffs[Sh::NB * 9];
  double norm[Sh::NB];
  double psi[Sh::LB * Sh::NQ * Sh::NB];
  double kw[Sh::LB * Sh::NQ * kMaxKinds];
  double y[Sh::LB * Sh::NQ * 3];
  double rr[Sh::LB * Sh::NQ];
  double vals[4 * kMaxKinds * Sh::NB];  // children values (all 4)
  double acc[kMaxKinds * Sh::NB];
  double psi0[Sh::NB];   // basis at the node's preimage (shifted gradient rows)
  double hco[Sh::NB];    // mode 1: the patch's curvature coefficients
  double item[Sh::ITEM];
  double cverts[4 * 6];
  double cmind[4], cdiam[4];
  double red[kQuadThreads / 32];
  long long pair;
};

// evaluate leaves [c0, c0 + L) of sm.cverts into sm.vals[c], cmind, cdiam
template <int ORDER>
__device__ void eval_leaves(const QuadArgs& A, QuadSmem<ORDER>& sm, int c0, int L, bool duffy, bool self,
                            const double x[3], const double nx[3]) {
  using Sh = QuadShape<ORDER>;
  constexpr int NB = Sh::NB;
  const int nq = duffy ? A.nqd : A.nqs;
  const double* rule = duffy ? A.drule : A.srule;
  const int nk = A.nk;
  for (int idx = threadIdx.x; idx < L * nq; idx += blockDim.x) {
    const int l = idx / nq, q = idx - l * nq;
    const double* v = sm.cverts + 6 * (c0 + l);
    const double e1u = v[2] - v[0], e1v = v[3] - v[1], e2u = v[4] - v[0], e2v = v[5] - v[1];
    const double area2 = fabs(e1u * e2v - e1v * e2u);
    const double aq = rule[3 * q], bq = rule[3 * q + 1], wq = rule[3 * q + 2];
    double uu, vv;
    if (duffy) {
      const double du = (1.0 - bq) * e1u + bq * e2u, dv = (1.0 - bq) * e1v + bq * e2v;
      uu = v[0] + aq * du;
      vv = v[1] + aq * dv;
    } else {
      uu = v[0] + aq * e1u + bq * e2u;
      vv = v[1] + aq * e1v + bq * e2v;
    }
    const int base = l * Sh::NQ + q;
    // basis straight into shared memory (the dot products below read it
    // there anyway): keeps the register footprint low enough for 2 CTAs/SM
    double* psi = sm.psi + base * NB;
    koornwinder_km<ORDER>(uu, vv, sm.norm, psi);
    double g[9];
#pragma unroll
    for (int c = 0; c < 9; ++c) g[c] = 0.0;
#pragma unroll 4
    for (int b = 0; b < NB; ++b) {
      const double pb = psi[b];
#pragma unroll
      for (int c = 0; c < 9; ++c) g[c] += pb * sm.coeffs[9 * b + c];
    }
    const double cr0 = g[4] * g[8] - g[5] * g[7];
    const double cr1 = g[5] * g[6] - g[3] * g[8];
    const double cr2 = g[3] * g[7] - g[4] * g[6];
    const double jac = sqrt(cr0 * cr0 + cr1 * cr1 + cr2 * cr2);
    const double ny0 = cr0 / jac, ny1 = cr1 / jac, ny2 = cr2 / jac;
    const double r0 = x[0] - g[0], r1 = x[1] - g[1], r2 = x[2] - g[2];
    double rr = r0 * r0 + r1 * r1 + r2 * r2;
    if (rr < 1e-280) rr = 1e-280;
    const double invr = 1.0 / sqrt(rr);
    const double invr3 = invr / rr;
    const double w = wq * area2 * jac;
    if (A.mode == 1) {
      // _pv_integrand (quadrature.py:252-274): 2H G n_y and (D kernel) n_y
      double hc = 0.0;
      for (int b = 0; b < NB; ++b) hc += psi[b] * sm.hco[b];
      const double gk = invr / kFourPi;
      const double dker = (r0 * ny0 + r1 * ny1 + r2 * ny2) / (rr * sqrt(rr)) / kFourPi;
      const double c = 2.0 * hc * gk * w, dw = dker * w;
      double* kwp = sm.kw + base * kMaxKinds;
      kwp[0] = c * ny0;
      kwp[1] = c * ny1;
      kwp[2] = c * ny2;
      kwp[3] = dw * ny0;
      kwp[4] = dw * ny1;
      kwp[5] = dw * ny2;
    } else
    for (int k = 0; k < nk; ++k) {
      double ker;
      switch (A.codes[k]) {
        case LB_KIND_S: ker = invr / kFourPi; break;
        case LB_KIND_D: ker = (r0 * ny0 + r1 * ny1 + r2 * ny2) * invr3 / kFourPi; break;
        case LB_KIND_SPRIME: ker = -(r0 * nx[0] + r1 * nx[1] + r2 * nx[2]) * invr3 / kFourPi; break;
        case LB_KIND_GRAD_S1: ker = -r0 * invr3 / kFourPi; break;
        case LB_KIND_GRAD_S2: ker = -r1 * invr3 / kFourPi; break;
        case LB_KIND_GRAD_S3: ker = -r2 * invr3 / kFourPi; break;
        default: {
          const double d0 = nx[0] - ny0, d1 = nx[1] - ny1, d2 = nx[2] - ny2;
          const double rnx = r0 * nx[0] + r1 * nx[1] + r2 * nx[2];
          const double rdn = r0 * d0 + r1 * d1 + r2 * d2;
          const double ndn = nx[0] * d0 + nx[1] * d1 + nx[2] * d2;
          ker = (3.0 * rnx * rdn / rr - ndn) * invr3 / kFourPi;
        }
      }
      sm.kw[base * kMaxKinds + k] = ker * w;
    }
    sm.y[3 * base] = g[0];
    sm.y[3 * base + 1] = g[1];
    sm.y[3 * base + 2] = g[2];
    sm.rr[base] = rr;
  }
  __syncthreads();
  // basis-weighted sums: vals[c][k][b] = sum_q kw[q][k] psi[q][b] (gradient
  // kinds on the self patch use the shifted basis psi - psi0,
  // _leafeval.py:172-174); mode 1: plain sums of the 6 PV components
  const int nbv = A.mode == 1 ? 1 : NB;
  for (int o = threadIdx.x; o < L * nk * nbv; o += blockDim.x) {
    const int l = o / (nk * nbv), kb = o - l * nk * nbv, k = kb / nbv, b = kb - k * nbv;
    const double* kwp = sm.kw + l * Sh::NQ * kMaxKinds + k;
    double s = 0.0;
    if (A.mode == 1) {
      for (int q = 0; q < nq; ++q) s += kwp[q * kMaxKinds];
    } else {
      const double* pp = sm.psi + l * Sh::NQ * NB + b;
      if (self && is_grad(A.codes[k])) {
        const double p0 = sm.psi0[b];
        for (int q = 0; q < nq; ++q) s += kwp[q * kMaxKinds] * (pp[q * NB] - p0);
      } else {
        for (int q = 0; q < nq; ++q) s += kwp[q * kMaxKinds] * pp[q * NB];
      }
    }
    sm.vals[((c0 + l) * kMaxKinds + k) * NB + b] = s;
  }
  // distance to the target and leaf diameter (_leafeval.py:137-190): one warp per leaf
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (warp < L) {
    const double* yy = sm.y + 3 * warp * Sh::NQ;
    const double* rp = sm.rr + warp * Sh::NQ;
    double md = 1e300, c0s = 0.0, c1s = 0.0, c2s = 0.0;
    for (int q = lane; q < nq; q += 32) {
      md = fmin(md, rp[q]);
    }
    // centroid: ordered sum by lane 0 keeps it deterministic
    if (lane == 0) {
      for (int q = 0; q < nq; ++q) {
        c0s += yy[3 * q];
        c1s += yy[3 * q + 1];
        c2s += yy[3 * q + 2];
      }
      c0s /= nq;
      c1s /= nq;
      c2s /= nq;
    }
    c0s = __shfl_sync(0xffffffffu, c0s, 0);
    c1s = __shfl_sync(0xffffffffu, c1s, 0);
    c2s = __shfl_sync(0xffffffffu, c2s, 0);
    double dm = 0.0;
    for (int q = lane; q < nq; q += 32) {
      const double t0 = yy[3 * q] - c0s, t1 = yy[3 * q + 1] - c1s, t2 = yy[3 * q + 2] - c2s;
      dm = fmax(dm, t0 * t0 + t1 * t1 + t2 * t2);
    }
    for (int o = 16; o > 0; o >>= 1) {
      md = fmin(md, __shfl_xor_sync(0xffffffffu, md, o));
      dm = fmax(dm, __shfl_xor_sync(0xffffffffu, dm, o));
    }
    if (lane == 0) {
      sm.cmind[c0 + warp] = sqrt(md);
      sm.cdiam[c0 + warp] = 2.0 * sqrt(dm);
    }
  }
  __syncthreads();
}

template <int ORDER>
__global__ void __launch_bounds__(kQuadThreads, 2) quad_pairs_kernel(QuadArgs A) {
  using Sh = QuadShape<ORDER>;
  constexpr int NB = Sh::NB;
  constexpr int ITEM = Sh::ITEM;
  extern __shared__ __align__(16) unsigned char smraw[];
  QuadSmem<ORDER>& sm = *reinterpret_cast<QuadSmem<ORDER>*>(smraw);
  const int nk = A.nk;
  const int nbv = A.mode == 1 ? 1 : NB;
  const int nkb = nk * nbv;
  bool any_grad = false;
  for (int k = 0; k < nk; ++k) any_grad |= A.mode == 0 && is_grad(A.codes[k]);
  double* stack = A.stack + (int64_t)blockIdx.x * kStackItems * ITEM;
  for (int i = threadIdx.x; i < NB; i += blockDim.x) sm.norm[i] = A.norm[i];
  for (;;) {
    if (threadIdx.x == 0) sm.pair = (long long)atomicAdd(A.next, 1ull);
    __syncthreads();
    const long long pair = sm.pair;
    if (pair >= A.npairs) break;
    const int64_t t = A.pair_tgt[pair];
    const int64_t p = A.pair_pat[pair];
    const bool self = A.node_patch[t] == p;
    const double x[3] = {A.nodes[3 * t], A.nodes[3 * t + 1], A.nodes[3 * t + 2]};
    const double nx[3] = {A.normals[3 * t], A.normals[3 * t + 1], A.normals[3 * t + 2]};
    for (int i = threadIdx.x; i < NB * 9; i += blockDim.x) sm.coeffs[i] = A.coeffs[p * NB * 9 + i];
    for (int i = threadIdx.x; i < nkb; i += blockDim.x) sm.acc[i] = 0.0;
    if (A.mode == 1)
      for (int i = threadIdx.x; i < NB; i += blockDim.x) sm.hco[i] = A.hcoeff[p * NB + i];
    // roots (quadrature.py:548-556): self -> 3 Duffy triangles at the node's
    // preimage, else the whole reference triangle
    const int nroot = self ? 3 : 1;
    if (threadIdx.x == 0) {
      const double corners[6] = {0.0, 0.0, 1.0, 0.0, 0.0, 1.0};
      if (self) {
        const double u0 = A.node_uv[2 * t], v0 = A.node_uv[2 * t + 1];
        for (int k = 0; k < 3; ++k) {
          double* cv = sm.cverts + 6 * k;
          cv[0] = u0;
          cv[1] = v0;
          cv[2] = corners[2 * k];
          cv[3] = corners[2 * k + 1];
          cv[4] = corners[2 * ((k + 1) % 3)];
          cv[5] = corners[2 * ((k + 1) % 3) + 1];
        }
      } else {
        for (int c = 0; c < 6; ++c) sm.cverts[c] = corners[c];
      }
      if (self && any_grad) koornwinder_km<ORDER>(A.node_uv[2 * t], A.node_uv[2 * t + 1], sm.norm, sm.psi0);
    }
    __syncthreads();
    // in batches of LB leaves (orders 8-9 hold 2 leaves' basis tables, a
    // self pair has 3 Duffy roots)
    for (int c0 = 0; c0 < nroot; c0 += Sh::LB) {
      eval_leaves<ORDER>(A, sm, c0, min(Sh::LB, nroot - c0), self, self, x, nx);
    }
    // push the roots (reverse order: the first root is refined first)
    int sp = 0;
    for (int r = nroot - 1; r >= 0; --r) {
      double* it = stack + (int64_t)sp * ITEM;
      for (int i = threadIdx.x; i < 10 + nkb; i += blockDim.x) {
        double val;
        if (i < 6) val = sm.cverts[6 * r + i];
        else if (i == 6) val = self ? 1.0 : 0.0;
        else if (i == 7) val = 0.0;
        else if (i == 8) val = sm.cmind[r];
        else if (i == 9) val = sm.cdiam[r];
        else val = sm.vals[(r * kMaxKinds + (i - 10) / nbv) * NB + (i - 10) % nbv];
        it[i] = val;
      }
      ++sp;
    }
    bool failed = false;
    while (sp > 0) {
      __syncthreads();
      // pop
      --sp;
      {
        const double* it = stack + (int64_t)sp * ITEM;
        for (int i = threadIdx.x; i < 10 + nkb; i += blockDim.x) sm.item[i] = it[i];
      }
      __syncthreads();
      const bool duffy = sm.item[6] != 0.0;
      const int depth = (int)sm.item[7];
      if (depth >= kMaxDepth) {
        if (threadIdx.x == 0) {
          atomicExch(A.status, 1);
          *A.bad_pair = pair;
        }
        failed = true;
        break;
      }
      // children (quadrature.py:337-386)
      const double* v = sm.item;
      const int nch = duffy ? 2 : 4;
      if (threadIdx.x == 0) {
        const double m12u = 0.5 * (v[2] + v[4]), m12v = 0.5 * (v[3] + v[5]);
        double* c = sm.cverts;
        if (duffy) {
          const double cv[12] = {v[0], v[1], v[2], v[3], m12u, m12v, v[0], v[1], m12u, m12v, v[4], v[5]};
          for (int i = 0; i < 12; ++i) c[i] = cv[i];
        } else {
          const double m01u = 0.5 * (v[0] + v[2]), m01v = 0.5 * (v[1] + v[3]);
          const double m20u = 0.5 * (v[4] + v[0]), m20v = 0.5 * (v[5] + v[1]);
          const double cv[24] = {v[0], v[1], m01u, m01v, m20u, m20v,   m01u, m01v, v[2], v[3], m12u, m12v,
                                 m20u, m20v, m12u, m12v, v[4], v[5],   m01u, m01v, m12u, m12v, m20u, m20v};
          for (int i = 0; i < 24; ++i) c[i] = cv[i];
        }
      }
      __syncthreads();
      for (int c0 = 0; c0 < nch; c0 += Sh::LB) {
        eval_leaves<ORDER>(A, sm, c0, min(Sh::LB, nch - c0), duffy, self, x, nx);
      }
      if (A.stats && threadIdx.x == 0) {
        atomicAdd(A.stats, 1ull);
        atomicAdd(A.stats + 1, (unsigned long long)nch);
      }
      // fine = sum of the children; err = max |fine - vals|
      double e = 0.0;
      for (int i = threadIdx.x; i < nkb; i += blockDim.x) {
        const int k = i / nbv, b = i - k * nbv;
        double f = 0.0;
        for (int c = 0; c < nch; ++c) f += sm.vals[(c * kMaxKinds + k) * NB + b];
        e = fmax(e, fabs(f - sm.item[10 + i]));
      }
      for (int o = 16; o > 0; o >>= 1) e = fmax(e, __shfl_xor_sync(0xffffffffu, e, o));
      if ((threadIdx.x & 31) == 0) sm.red[threadIdx.x >> 5] = e;
      __syncthreads();
      double err = 0.0;
      for (int w = 0; w < kQuadThreads / 32; ++w) err = fmax(err, sm.red[w]);
      const double e1u = v[2] - v[0], e1v = v[3] - v[1], e2u = v[4] - v[0], e2v = v[5] - v[1];
      const double frac = fabs(e1u * e2v - e1v * e2u);
      const double tol = 0.1 * A.eps * fmax(sqrt(frac), 1e-3);
      const bool force = !self && (sm.item[9] > 0.8 * sm.item[8]);
      const bool ok = (err <= tol) && !force;
      if (ok) {
        for (int i = threadIdx.x; i < nkb; i += blockDim.x) {
          const int k = i / nbv, b = i - k * nbv;
          double f = 0.0;
          for (int c = 0; c < nch; ++c) f += sm.vals[(c * kMaxKinds + k) * NB + b];
          sm.acc[i] += f;
        }
      } else {
        // push children, last child first so child 0 is refined next
        for (int c = nch - 1; c >= 0; --c) {
          double* it = stack + (int64_t)sp * ITEM;
          for (int i = threadIdx.x; i < 10 + nkb; i += blockDim.x) {
            double val;
            if (i < 6) val = sm.cverts[6 * c + i];
            else if (i == 6) val = duffy ? 1.0 : 0.0;
            else if (i == 7) val = (double)(depth + 1);
            else if (i == 8) val = sm.cmind[c];
            else if (i == 9) val = sm.cdiam[c];
            else val = sm.vals[(c * kMaxKinds + (i - 10) / nbv) * NB + (i - 10) % nbv];
            it[i] = val;
          }
          ++sp;
        }
        if (sp > kStackItems - 4) {  // cannot happen below the depth cap
          if (threadIdx.x == 0) {
            atomicExch(A.status, 2);
            *A.bad_pair = pair;
          }
          failed = true;
          break;
        }
      }
    }
    __syncthreads();
    if (failed) break;
    double* out = A.acc + pair * (int64_t)nkb;
    for (int i = threadIdx.x; i < nkb; i += blockDim.x) out[i] = sm.acc[i];
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// assembly

struct AsmArgs {
  int nb, nk, nbo;
  int codes[kMaxKinds];
  const double* acc;          // (npairs, nk, nb) k-major
  const int32_t* kmajor_perm; // (nb): degree-major column j <- k-major perm[j]
  const double* vinv;         // (nb, nb)
  const double* over_interp;  // (nbo, nb)
  const double* nodes, *normals;
  const double* over_nodes, *over_normals, *over_weights;  // patch-major
  const int64_t* pair_tgt;
  const int32_t* pair_pat;
  const int64_t* pair_pos;    // CSR value offset of the pair's nb columns
  int64_t npairs;
  double* vals[kMaxKinds];    // CSR value arrays, one per kind
  const int64_t* node_patch;  // self-pair test for the PV term
  const double* pv;           // (N, 3) PV constants of grad S over the own patch, or null
  const double* pvrow;        // (N, nb) interpolation row at the node's preimage
};

__global__ void __launch_bounds__(128) corr_assemble_kernel(AsmArgs A) {
  extern __shared__ double sa[];
  const int nb = A.nb, nk = A.nk, nbo = A.nbo;
  double* kwo = sa;               // nbo * nk
  double* accd = sa + nbo * nk;   // nk * nb (degree-major)
  for (int64_t pair = blockIdx.x; pair < A.npairs; pair += gridDim.x) {
    const int64_t t = A.pair_tgt[pair];
    const int64_t p = A.pair_pat[pair];
    const double x0 = A.nodes[3 * t], x1 = A.nodes[3 * t + 1], x2 = A.nodes[3 * t + 2];
    const double n0 = A.normals[3 * t], n1 = A.normals[3 * t + 1], n2 = A.normals[3 * t + 2];
    __syncthreads();
    // smooth oversampled rule (quadrature.py:593-610, kernels as _kernel_values 115-136)
    for (int q = threadIdx.x; q < nbo; q += blockDim.x) {
      const int64_t j = p * nbo + q;
      const double r0 = x0 - A.over_nodes[3 * j], r1 = x1 - A.over_nodes[3 * j + 1],
                   r2 = x2 - A.over_nodes[3 * j + 2];
      const double ny0 = A.over_normals[3 * j], ny1 = A.over_normals[3 * j + 1], ny2 = A.over_normals[3 * j + 2];
      const double rr = r0 * r0 + r1 * r1 + r2 * r2;
      const double invr3 = 1.0 / (rr * sqrt(rr));
      const double w = A.over_weights[j];
      for (int k = 0; k < nk; ++k) {
        double ker;
        switch (A.codes[k]) {
          case LB_KIND_S: ker = invr3 * rr / kFourPi; break;
          case LB_KIND_D: ker = (r0 * ny0 + r1 * ny1 + r2 * ny2) * invr3 / kFourPi; break;
          case LB_KIND_SPRIME: ker = -(r0 * n0 + r1 * n1 + r2 * n2) * invr3 / kFourPi; break;
          case LB_KIND_GRAD_S1: ker = -r0 * invr3 / kFourPi; break;
          case LB_KIND_GRAD_S2: ker = -r1 * invr3 / kFourPi; break;
          case LB_KIND_GRAD_S3: ker = -r2 * invr3 / kFourPi; break;
          default: {
            const double d0 = n0 - ny0, d1 = n1 - ny1, d2 = n2 - ny2;
            const double rnx = r0 * n0 + r1 * n1 + r2 * n2;
            const double rdn = r0 * d0 + r1 * d1 + r2 * d2;
            const double ndn = n0 * d0 + n1 * d1 + n2 * d2;
            ker = (3.0 * rnx * rdn / rr - ndn) * invr3 / kFourPi;
          }
        }
        kwo[q * nk + k] = ker * w;
      }
    }
    for (int i = threadIdx.x; i < nk * nb; i += blockDim.x) {
      const int k = i / nb, j = i - k * nb;
      accd[i] = A.acc[(pair * nk + k) * nb + A.kmajor_perm[j]];
    }
    __syncthreads();
    const int64_t pos = A.pair_pos[pair];
    for (int i = threadIdx.x; i < nk * nb; i += blockDim.x) {
      const int k = i / nb, b = i - k * nb;
      double rows = 0.0;
      for (int j = 0; j < nb; ++j) rows += accd[k * nb + j] * A.vinv[j * nb + b];
      double over = 0.0;
      for (int q = 0; q < nbo; ++q) over += kwo[q * nk + k] * A.over_interp[q * nb + b];
      const int code = A.codes[k];
      if (A.pv && is_grad(code) && A.node_patch[t] == p)  // quadrature.py:685-688
        rows += A.pv[3 * t + (code - LB_KIND_GRAD_S1)] * A.pvrow[t * nb + b];
      A.vals[k][pos + b] = rows - over;
    }
  }
}

// ---------------------------------------------------------------------------
// principal-value constants (quadrature.py:424-498, 562-590)

constexpr int kBndStack = 64;

// line integral of G(x, y) nu around the own patch (_boundary_g_integral):
// one warp per (target, edge), adaptive bisection of Gauss panels
template <int ORDER>
__global__ void __launch_bounds__(128) pv_boundary_kernel(const double* __restrict__ coeffs,
                                                          const double* __restrict__ nodes,
                                                          const int64_t* __restrict__ node_patch,
                                                          const double* __restrict__ norm,
                                                          const double* __restrict__ gauss, int ng, int64_t n,
                                                          double eps, double* __restrict__ bnd, int* status) {
  constexpr int NB = ORDER * (ORDER + 1) / 2;
  __shared__ double sh[4][32][5];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t item = (int64_t)blockIdx.x * 4 + wib;
  if (item >= 3 * n) return;
  const int64_t t = item / 3;
  const int e = (int)(item % 3);
  const int64_t p = node_patch[t];
  const double* cf = coeffs + p * NB * 9;
  const double x0 = nodes[3 * t], x1 = nodes[3 * t + 1], x2 = nodes[3 * t + 2];
  const double cu[3] = {0.0, 1.0, 0.0}, cv[3] = {0.0, 0.0, 1.0};
  const double e0u = cu[e], e0v = cv[e], e1u = cu[(e + 1) % 3], e1v = cv[(e + 1) % 3];
  const double du = e1u - e0u, dv = e1v - e0v;
  double (*S)[5] = sh[wib];
  // evaluate panel [a, b] on lanes [h * ng, h * ng + ng): returns (vals, dist, plen) on all lanes
  auto panel = [&](double a, double b, int h, double out[5]) {
    if (lane >= h * ng && lane < (h + 1) * ng) {
      const int q = lane - h * ng;
      const double tl = a + (b - a) * gauss[2 * q];
      const double uu = e0u + tl * du, vv = e0v + tl * dv;
      double psi[NB];
      {
        double buf[NB];
        koornwinder_km<ORDER>(uu, vv, norm, buf);
#pragma unroll
        for (int i = 0; i < NB; ++i) psi[i] = buf[i];
      }
      double g[9];
#pragma unroll
      for (int c = 0; c < 9; ++c) g[c] = 0.0;
#pragma unroll
      for (int bb = 0; bb < NB; ++bb) {
#pragma unroll
        for (int c = 0; c < 9; ++c) g[c] += psi[bb] * cf[9 * bb + c];
      }
      const double tv0 = g[3] * du + g[6] * dv, tv1 = g[4] * du + g[7] * dv, tv2 = g[5] * du + g[8] * dv;
      const double tlen = sqrt(tv0 * tv0 + tv1 * tv1 + tv2 * tv2);
      const double th0 = tv0 / tlen, th1 = tv1 / tlen, th2 = tv2 / tlen;
      const double c0 = g[4] * g[8] - g[5] * g[7], c1 = g[5] * g[6] - g[3] * g[8], c2 = g[3] * g[7] - g[4] * g[6];
      const double cn = sqrt(c0 * c0 + c1 * c1 + c2 * c2);
      const double n0 = c0 / cn, n1 = c1 / cn, n2 = c2 / cn;
      const double nu0 = th1 * n2 - th2 * n1, nu1 = th2 * n0 - th0 * n2, nu2 = th0 * n1 - th1 * n0;
      const double r0 = x0 - g[0], r1 = x1 - g[1], r2 = x2 - g[2];
      const double gk = 1.0 / (kFourPi * sqrt(r0 * r0 + r1 * r1 + r2 * r2));
      const double sc = gk * ((b - a) * gauss[2 * q + 1]) * tlen;
      S[lane][0] = sc * nu0;
      S[lane][1] = sc * nu1;
      S[lane][2] = sc * nu2;
      S[lane][3] = tlen;
      S[lane][4] = sqrt(r0 * r0 + r1 * r1 + r2 * r2);  // |x - y_q|
    }
    __syncwarp();
    double v0 = 0.0, v1 = 0.0, v2 = 0.0, tsum = 0.0;
    for (int q = 0; q < ng; ++q) {  // ordered sums: deterministic
      v0 += S[h * ng + q][0];
      v1 += S[h * ng + q][1];
      v2 += S[h * ng + q][2];
      tsum += S[h * ng + q][3];
    }
    out[0] = v0;
    out[1] = v1;
    out[2] = v2;
    out[3] = S[h * ng + ng / 2][4];          // distance to the middle node
    out[4] = tsum / ng * (b - a);             // panel length
    __syncwarp();
  };
  double st[kBndStack][6];  // a, b, v0, v1, v2 (dist/plen kept separately)
  double sdist[kBndStack], splen[kBndStack];
  int sdep[kBndStack];
  double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
  double r[5];
  panel(0.0, 1.0, 0, r);
  int sp = 0;
  st[0][0] = 0.0;
  st[0][1] = 1.0;
  st[0][2] = r[0];
  st[0][3] = r[1];
  st[0][4] = r[2];
  sdist[0] = r[3];
  splen[0] = r[4];
  sdep[0] = 0;
  sp = 1;
  while (sp > 0) {
    --sp;
    const double a = st[sp][0], b = st[sp][1];
    const double pv0 = st[sp][2], pv1 = st[sp][3], pv2 = st[sp][4], plen = splen[sp];
    const int dep = sdep[sp];
    if (dep >= kMaxDepth || sp >= kBndStack - 2) {
      if (lane == 0) atomicExch(status, 3);
      return;
    }
    const double mid = 0.5 * (a + b);
    double r1[5], r2[5];
    // both halves at once: lanes [0, ng) and [ng, 2 ng)
    {
      double o1[5], o2[5];
      panel(a, mid, 0, o1);
      panel(mid, b, 1, o2);
      for (int i = 0; i < 5; ++i) { r1[i] = o1[i]; r2[i] = o2[i]; }
    }
    const double f0 = r1[0] + r2[0], f1 = r1[1] + r2[1], f2 = r1[2] + r2[2];
    const double err = fmax(fabs(f0 - pv0), fmax(fabs(f1 - pv1), fabs(f2 - pv2)));
    const bool force = plen > 0.8 * fmin(r1[3], r2[3]);
    const bool ok = err <= 0.1 * eps * fmax(sqrt(b - a), 1e-3) && !force;
    if (ok) {
      acc0 += f0;
      acc1 += f1;
      acc2 += f2;
    } else {
      st[sp][0] = mid; st[sp][1] = b; st[sp][2] = r2[0]; st[sp][3] = r2[1]; st[sp][4] = r2[2];
      sdist[sp] = r2[3]; splen[sp] = r2[4]; sdep[sp] = dep + 1; ++sp;
      st[sp][0] = a; st[sp][1] = mid; st[sp][2] = r1[0]; st[sp][3] = r1[1]; st[sp][4] = r1[2];
      sdist[sp] = r1[3]; splen[sp] = r1[4]; sdep[sp] = dep + 1; ++sp;
    }
  }
  if (lane == 0) {
    bnd[t * 9 + e * 3] = acc0;
    bnd[t * 9 + e * 3 + 1] = acc1;
    bnd[t * 9 + e * 3 + 2] = acc2;
  }
}

// pv = -(boundary + curvature term + double-layer term) (quadrature.py:590)
// and the interpolation row psi(uv0) @ vinv (quadrature.py:684)
template <int ORDER>
__global__ void pv_combine_kernel(const double* __restrict__ bnd, const double* __restrict__ pvacc,
                                  const double* __restrict__ node_uv, const double* __restrict__ norm,
                                  const int32_t* __restrict__ perm, const double* __restrict__ vinv, int64_t n,
                                  double* __restrict__ pv, double* __restrict__ pvrow) {
  constexpr int NB = ORDER * (ORDER + 1) / 2;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  for (int c = 0; c < 3; ++c) {
    const double boundary = (bnd[t * 9 + c] + bnd[t * 9 + 3 + c]) + bnd[t * 9 + 6 + c];
    pv[3 * t + c] = -((boundary + pvacc[6 * t + c]) + pvacc[6 * t + 3 + c]);
  }
  double psi[NB];
  koornwinder_km<ORDER>(node_uv[2 * t], node_uv[2 * t + 1], norm, psi);
  for (int b = 0; b < NB; ++b) {
    double s = 0.0;
    for (int j = 0; j < NB; ++j) s += psi[perm[j]] * vinv[j * NB + b];
    pvrow[t * NB + b] = s;
  }
}

template <int ORDER>
int launch_quad(const QuadArgs& A, int grid, cudaStream_t st);

template <int ORDER>
int launch_pv(const lb_corr_build_desc* d, QuadArgs A, int grid, Scratch& s_pv, Scratch& s_row,
              cudaStream_t st) {
  constexpr int NB = ORDER * (ORDER + 1) / 2;
  const int64_t n = d->n;
  Scratch s_tgt, s_pat, s_acc, s_bnd;
  LB_TRY(s_tgt.alloc(sizeof(int64_t) * n, st));
  LB_TRY(s_pat.alloc(sizeof(int32_t) * n, st));
  LB_TRY(s_acc.alloc(sizeof(double) * 6 * n, st));
  LB_TRY(s_bnd.alloc(sizeof(double) * 9 * n, st));
  LB_TRY(s_pv.alloc(sizeof(double) * 3 * n, st));
  LB_TRY(s_row.alloc(sizeof(double) * NB * n, st));
  self_pairs_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d->node_patch, n, static_cast<int64_t*>(s_tgt.ptr),
                                                                static_cast<int32_t*>(s_pat.ptr));
  LB_CHECK_LAUNCH();
  // _pv_constants' adaptive part: 3 Duffy roots per target, 6 components
  A.mode = 1;
  A.nk = 6;
  A.hcoeff = d->hcoeff_km;
  A.pair_tgt = static_cast<int64_t*>(s_tgt.ptr);
  A.pair_pat = static_cast<int32_t*>(s_pat.ptr);
  A.npairs = n;
  A.acc = static_cast<double*>(s_acc.ptr);
  LB_CUDA(cudaMemsetAsync(A.next, 0, 8, st));
  LB_TRY(launch_quad<ORDER>(A, grid, st));
  pv_boundary_kernel<ORDER><<<(unsigned)ceil_div(3 * n, 4), 128, 0, st>>>(
      d->coeffs_km, d->nodes, d->node_patch, d->knorm, d->gauss, d->ng, n, d->eps,
      static_cast<double*>(s_bnd.ptr), A.status);
  LB_CHECK_LAUNCH();
  pv_combine_kernel<ORDER><<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(
      static_cast<double*>(s_bnd.ptr), static_cast<double*>(s_acc.ptr), d->node_uv, d->knorm, d->kmajor_perm,
      d->vinv, n, static_cast<double*>(s_pv.ptr), static_cast<double*>(s_row.ptr));
  LB_CHECK_LAUNCH();
  return LB_OK;
}

template <int ORDER>
int launch_quad(const QuadArgs& A, int grid, cudaStream_t st) {
  const size_t smem = sizeof(QuadSmem<ORDER>);
  LB_CUDA(cudaFuncSetAttribute(quad_pairs_kernel<ORDER>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  quad_pairs_kernel<ORDER><<<grid, kQuadThreads, smem, st>>>(A);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

template <int ORDER>
size_t quad_item_doubles() { return QuadShape<ORDER>::ITEM; }

}  // namespace
}  // namespace lb

using namespace lb;

extern "C" {

int lb_near_map_count(const double* nodes, int64_t n, const double* centers, const double* radii_eta,
                      int64_t npatches, const int64_t* node_patch, int32_t* counts, void* stream) {
  if (n < 0 || npatches <= 0) return fail(LB_ERR_SHAPE, "lb_near_map_count: bad sizes");
  if (n == 0) return LB_OK;
  if (!nodes || !centers || !radii_eta || !node_patch || !counts)
    return fail(LB_ERR_ARG, "lb_near_map_count: null pointer");
  near_kernel<false><<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(
      nodes, n, centers, radii_eta, npatches, node_patch, counts, nullptr, nullptr);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

int lb_near_map_fill(const double* nodes, int64_t n, const double* centers, const double* radii_eta,
                     int64_t npatches, const int64_t* node_patch, const int64_t* offsets, int32_t* patches,
                     void* stream) {
  if (n < 0 || npatches <= 0) return fail(LB_ERR_SHAPE, "lb_near_map_fill: bad sizes");
  if (n == 0) return LB_OK;
  if (!nodes || !centers || !radii_eta || !node_patch || !offsets || !patches)
    return fail(LB_ERR_ARG, "lb_near_map_fill: null pointer");
  near_kernel<true><<<(unsigned)ceil_div(n, 128), 128, 0, as_stream(stream)>>>(
      nodes, n, centers, radii_eta, npatches, node_patch, nullptr, offsets, patches);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

int lb_corrections_build(const lb_corr_build_desc* d, void* stream) {
  if (!d) return fail(LB_ERR_ARG, "lb_corrections_build: null descriptor");
  if (!(d->eps >= 1e-12 && d->eps <= 1e-3))
    return fail(LB_ERR_EPS, "eps must lie in [1e-12, 1e-3]");  // quadrature.py:670-671
  if (d->nk < 1 || d->nk > kMaxKinds) return fail(LB_ERR_ARG, "lb_corrections_build: nk must be in [1, 7]");
  for (int k = 0; k < d->nk; ++k) {
    const int c = d->kinds[k];
    if (c < 0 || c > 6) return fail(LB_ERR_KEY, "lb_corrections_build: unknown kind code");
    if (is_grad(c)) {
      if (!d->hcoeff_km || !d->gauss || d->ng < 1 || d->ng > 16 || d->n <= 0)
        return fail(LB_ERR_ARG, "lb_corrections_build: gradient kinds need hcoeff_km, gauss, ng and n");
    }
  }
  if (d->order < 2 || d->order > 9) return fail(LB_ERR_ARG, "lb_corrections_build: order must be in [2, 9]");
  const int nb = d->order * (d->order + 1) / 2;
  if (d->npairs == 0) return LB_OK;
  cudaStream_t st = as_stream(stream);
  QuadArgs A{};
  A.nb = nb;
  A.nk = d->nk;
  A.nqs = d->nqs;
  A.nqd = d->nqd;
  for (int k = 0; k < d->nk; ++k) A.codes[k] = d->kinds[k];
  A.eps = d->eps;
  A.coeffs = d->coeffs_km;
  A.nodes = d->nodes;
  A.normals = d->normals;
  A.node_uv = d->node_uv;
  A.node_patch = d->node_patch;
  A.pair_tgt = d->pair_tgt;
  A.pair_pat = d->pair_pat;
  A.npairs = d->npairs;
  A.srule = d->srule;
  A.drule = d->drule;
  A.norm = d->knorm;
  A.stats = reinterpret_cast<unsigned long long*>(d->stats);
  if (d->nqs > (d->order + 2) * (d->order + 2) || d->nqd > (d->order + 2) * (d->order + 2))
    return fail(LB_ERR_ARG, "lb_corrections_build: leaf rules larger than (order + 2)^2 points");
  // scratch: basis integrals, per-CTA item stacks, counters
  const int per_sm = 2;
  const int grid = sm_count() * per_sm;
  const size_t item = 10 + (size_t)kMaxKinds * nb;
  Scratch s_acc, s_stack, s_cnt;
  LB_TRY(s_acc.alloc(sizeof(double) * d->npairs * d->nk * nb, st));
  LB_TRY(s_stack.alloc(sizeof(double) * (size_t)grid * kStackItems * item, st));
  LB_TRY(s_cnt.alloc(64, st));
  LB_CUDA(cudaMemsetAsync(s_cnt.ptr, 0, 64, st));
  A.acc = static_cast<double*>(s_acc.ptr);
  A.stack = static_cast<double*>(s_stack.ptr);
  A.next = static_cast<unsigned long long*>(s_cnt.ptr);
  A.status = reinterpret_cast<int*>(static_cast<char*>(s_cnt.ptr) + 8);
  A.bad_pair = reinterpret_cast<long long*>(static_cast<char*>(s_cnt.ptr) + 16);
  switch (d->order) {
    case 2: LB_TRY(launch_quad<2>(A, grid, st)); break;
    case 3: LB_TRY(launch_quad<3>(A, grid, st)); break;
    case 4: LB_TRY(launch_quad<4>(A, grid, st)); break;
    case 5: LB_TRY(launch_quad<5>(A, grid, st)); break;
    case 6: LB_TRY(launch_quad<6>(A, grid, st)); break;
    case 7: LB_TRY(launch_quad<7>(A, grid, st)); break;
    case 8: LB_TRY(launch_quad<8>(A, grid, st)); break;
    default: LB_TRY(launch_quad<9>(A, grid, st)); break;
  }
  // principal-value constants for the gradient kinds (quadrature.py:679-688)
  bool any_grad = false;
  for (int k = 0; k < d->nk; ++k) any_grad |= is_grad(d->kinds[k]);
  Scratch s_pv, s_row;
  if (any_grad) {
    switch (d->order) {
      case 2: LB_TRY(launch_pv<2>(d, A, grid, s_pv, s_row, st)); break;
      case 3: LB_TRY(launch_pv<3>(d, A, grid, s_pv, s_row, st)); break;
      case 4: LB_TRY(launch_pv<4>(d, A, grid, s_pv, s_row, st)); break;
      case 5: LB_TRY(launch_pv<5>(d, A, grid, s_pv, s_row, st)); break;
      case 6: LB_TRY(launch_pv<6>(d, A, grid, s_pv, s_row, st)); break;
      case 7: LB_TRY(launch_pv<7>(d, A, grid, s_pv, s_row, st)); break;
      case 8: LB_TRY(launch_pv<8>(d, A, grid, s_pv, s_row, st)); break;
      default: LB_TRY(launch_pv<9>(d, A, grid, s_pv, s_row, st)); break;
    }
  }
  int flags[6] = {0, 0, 0, 0, 0, 0};
  LB_CUDA(cudaMemcpyAsync(flags, static_cast<char*>(s_cnt.ptr) + 8, 16, cudaMemcpyDeviceToHost, st));
  LB_CUDA(cudaStreamSynchronize(st));
  if (flags[0] == 3) return fail(LB_ERR_DEPTH, "boundary integral depth cap");  // quadrature.py:478-479
  if (flags[0] != 0) {
    long long bp = 0;
    std::memcpy(&bp, &flags[2], 8);
    return fail(LB_ERR_DEPTH, "adaptive integration exceeded depth 30; pair " + std::to_string(bp));
  }
  // assembly into the CSR values
  AsmArgs B{};
  B.nb = nb;
  B.nk = d->nk;
  B.nbo = d->nbo;
  for (int k = 0; k < d->nk; ++k) {
    B.codes[k] = d->kinds[k];
    B.vals[k] = d->values[k];
    if (!d->values[k]) return fail(LB_ERR_ARG, "lb_corrections_build: missing value array");
  }
  B.acc = A.acc;
  B.kmajor_perm = d->kmajor_perm;
  B.vinv = d->vinv;
  B.over_interp = d->over_interp;
  B.nodes = d->nodes;
  B.normals = d->normals;
  B.over_nodes = d->over_nodes;
  B.over_normals = d->over_normals;
  B.over_weights = d->over_weights;
  B.pair_tgt = d->pair_tgt;
  B.pair_pat = d->pair_pat;
  B.pair_pos = d->pair_pos;
  B.npairs = d->npairs;
  B.node_patch = d->node_patch;
  B.pv = any_grad ? static_cast<const double*>(s_pv.ptr) : nullptr;
  B.pvrow = any_grad ? static_cast<const double*>(s_row.ptr) : nullptr;
  const size_t smem = sizeof(double) * ((size_t)d->nbo * d->nk + (size_t)d->nk * nb);
  if (smem > 200 * 1024) return fail(LB_ERR_ARG, "lb_corrections_build: oversampled rule too large");
  LB_CUDA(cudaFuncSetAttribute(corr_assemble_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned ag = (unsigned)std::min<int64_t>(d->npairs, (int64_t)sm_count() * 16);
  corr_assemble_kernel<<<ag, 128, smem, st>>>(B);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

}  // extern "C"
