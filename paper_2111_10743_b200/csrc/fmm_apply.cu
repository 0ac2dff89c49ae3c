// FmmPlan.apply (fmm.py:784-990) on the B200.
//
//   gather   : charges/dipoles into Morton-sorted source order (one pass)
//   P2M      : surface: check potentials at the UC lattice of every source
//              leaf (pairwise kernel) then one DGEMM with pinv_up;
//              grid: Lagrange anterpolation kernel (charges + dipole terms)
//   M2M      : per (level, octant) DGEMM (surface) / separable 3x1-D kernel
//              (grid), children accumulated in octant order like fmm.py:853-871
//   M2L      : pairs grouped by CANONICAL offset across all levels: gather with
//              the inverse cube-symmetry permutation (and 1/h), ONE DGEMM with
//              the canonical matrix, deterministic per-target accumulation
//              through the forward permutation (no permuted matrix is ever
//              built; the reference spends most of a config-2 apply there)
//   X        : source leaves -> downward check points (pairwise kernel)
//   L2L      : per level DGEMM with pinv_dn (surface; grid: local = dcheck),
//              per (level, octant) DGEMM / separable kernel into the children
//   leaf     : grid L2T (value/grad/hess of the Chebyshev interpolant), then ONE
//              pairwise kernel per target leaf over U-list sources, the own
//              downward-equivalent charges (surface) and W-list equivalent
//              charges, exactly the fused leaf stage of fmm.py:937-988
//   scatter  : sorted targets -> reference layout (pot, grad, full hess)
//
// Every GEMM-shaped stage (surface P2M / M2M / L2L, the M2L factors) runs on
// the FP64 tensor cores through dgemm_cols.cuh (DMMA 8x8x4, gathers and
// scatters fused into the operand loads and the epilogue); no library GEMM.
#include <cub/cub.cuh>

#include <algorithm>
#include <climits>
#include <climits>
#include <cmath>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <map>
#include <string>
#include <tuple>
#include <vector>

#include "dgemm_cols.cuh"
#include "fmm_plan.h"
#include "lb_common.cuh"
#include "m2l_first.cuh"
#include "m2l_fused.cuh"
#include "ozaki.cuh"
#include "p2p_core.cuh"

namespace lb {

constexpr int kStages = 8;  // p2m m2m m2l x l2l l2t leaf scatter (+ total)

#define LB_DG(expr)                                                                \
  do {                                                                             \
    cudaError_t _e = (expr);                                                       \
    if (_e != cudaSuccess)                                                         \
      return fail(LB_ERR_CUDA, std::string("dgemm_cols (") + __FILE__ + ":" +      \
                                   std::to_string(__LINE__) + "): " + cudaGetErrorString(_e)); \
  } while (0)

// ---------------------------------------------------------------------------
// small device helpers

__global__ void gather_sources_kernel(const double* __restrict__ charges,
                                      const double* __restrict__ dipoles,
                                      const int64_t* __restrict__ src_sorted, int64_t ns, int nd,
                                      int d0, uint32_t cmask, uint32_t dmask, double* __restrict__ cs,
                                      double* __restrict__ vs) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= ns) return;
  const int64_t o = src_sorted[p];
  for (int l = 0; l < nd; ++l) {
    const int d = d0 + l;
    cs[(int64_t)l * ns + p] = ((cmask >> d) & 1u) ? charges[(int64_t)d * ns + o] : 0.0;
    const bool on = (dmask >> d) & 1u;
    for (int k = 0; k < 3; ++k)
      vs[((int64_t)l * ns + p) * 3 + k] = on ? dipoles[((int64_t)d * ns + o) * 3 + k] : 0.0;
  }
}

// ---------------------------------------------------------------------------
// potentials at lattice points from real sources (P2M check, X list)

// out[(box_col*nd + l)*nrep + i] (+)= scale * sum_j pot_l(x_i; sources of the
// listed leaves).  Points x_i = center(box) + fac*half(box)*pts[i].  Every
// thread holds LPT lattice points in registers (729 grid points = 6 per
// thread of 128) and the sources stream through shared memory ONCE per box:
// LPT independent pair chains per source (ILP) and 1/LPT of the tile loads
// and barriers of a one-point-per-thread pass.
constexpr int kLatBT = 128;

// DM: compile-time mask of the chunk's densities that carry dipoles (the A3
// projected call has them on its first density only: the second skips the
// dipole dot product instead of multiplying zeros -- the sums are the same
// bit for bit, fma(0, x, acc) = acc)
template <int ND, int kLatLPT, unsigned DM>
__global__ void __launch_bounds__(kLatBT) lattice_pot_kernel(
    const int64_t* __restrict__ boxes, const int64_t* __restrict__ src_off,
    const int64_t* __restrict__ src_boxes, int single, const double* __restrict__ bctr,
    const double* __restrict__ bhalf, const int64_t* __restrict__ bsrc,
    const double* __restrict__ spos, const double* __restrict__ cs, const double* __restrict__ vs,
    int64_t ns, int dm, const double* __restrict__ pts, int nrep, double fac, int scale_by_h,
    double* __restrict__ out, int out_by_box, int add) {
  constexpr int TS = 64;
  constexpr int W = 3 + 4 * ND;
  __shared__ double sh[TS * W];
  const int64_t bi = blockIdx.x;
  const int64_t b = boxes[bi];
  const double h = bhalf[b];
  const double cx = bctr[3 * b], cy = bctr[3 * b + 1], cz = bctr[3 * b + 2];
  const int64_t lb = single ? bi : src_off[bi];
  const int64_t le = single ? bi + 1 : src_off[bi + 1];
  for (int i0 = 0; i0 < nrep; i0 += kLatBT * kLatLPT) {  // one round for nrep <= 768
    double px[kLatLPT], py[kLatLPT], pz[kLatLPT], acc[kLatLPT][ND];
#pragma unroll
    for (int j = 0; j < kLatLPT; ++j) {
      const int i = i0 + j * kLatBT + threadIdx.x;
      const bool in = i < nrep;
      px[j] = in ? cx + fac * h * pts[3 * i] : 0.0;
      py[j] = in ? cy + fac * h * pts[3 * i + 1] : 0.0;
      pz[j] = in ? cz + fac * h * pts[3 * i + 2] : 0.0;
#pragma unroll
      for (int l = 0; l < ND; ++l) acc[j][l] = 0.0;
    }
    for (int64_t q = lb; q < le; ++q) {
      const int64_t sb = single ? b : src_boxes[q];
      const int64_t s0 = bsrc[2 * sb], s1 = bsrc[2 * sb + 1];
      for (int64_t t0 = s0; t0 < s1; t0 += TS) {
        const int n = (int)min((int64_t)TS, s1 - t0);
        __syncthreads();
        for (int k = threadIdx.x; k < n; k += kLatBT) {
          const int64_t j = t0 + k;
          double* r = sh + k * W;
          r[0] = spos[3 * j];
          r[1] = spos[3 * j + 1];
          r[2] = spos[3 * j + 2];
#pragma unroll
          for (int l = 0; l < ND; ++l) {
            r[3 + l] = cs[(int64_t)l * ns + j];
            if ((DM >> l) & 1u) {
              r[3 + ND + 3 * l] = vs[((int64_t)l * ns + j) * 3];
              r[4 + ND + 3 * l] = vs[((int64_t)l * ns + j) * 3 + 1];
              r[5 + ND + 3 * l] = vs[((int64_t)l * ns + j) * 3 + 2];
            }
          }
        }
        __syncthreads();
        for (int k = 0; k < n; ++k) {
          const double* r = sh + k * W;
#pragma unroll
          for (int j = 0; j < kLatLPT; ++j) {
            const double r0 = px[j] - r[0], r1 = py[j] - r[1], r2 = pz[j] - r[2];
            const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
            const double invr = inv_sqrt_skip(rr);
            double invr3 = 0.0;
            if constexpr (DM != 0u) invr3 = invr * invr * invr;
#pragma unroll
            for (int l = 0; l < ND; ++l) {
              if ((DM >> l) & 1u) {
                const double vr = fma(r[5 + ND + 3 * l], r2, fma(r[4 + ND + 3 * l], r1, r[3 + ND + 3 * l] * r0));
                acc[j][l] = fma(r[3 + l], invr, fma(vr, invr3, acc[j][l]));
              } else {
                acc[j][l] = fma(r[3 + l], invr, acc[j][l]);
              }
            }
          }
        }
      }
    }
    const double sc = scale_by_h ? h : 1.0;
    const int64_t col = out_by_box ? b : bi;
#pragma unroll
    for (int j = 0; j < kLatLPT; ++j) {
      const int i = i0 + j * kLatBT + threadIdx.x;
      if (i < nrep) {
#pragma unroll
        for (int l = 0; l < ND; ++l) {
          double* o = out + (col * ND + l) * (int64_t)nrep + i;
          *o = add ? *o + sc * acc[j][l] : sc * acc[j][l];
        }
      }
    }
  }
}

// lattice points per thread sized to the lattice (296 surface points: 3;
// 488: 4; 729 grid points: 6; larger lattices loop); dipole mask exact for
// one or two densities, all-or-none for more
template <int ND, unsigned DM, class... A>
int launch_lattice_dm(unsigned grid, cudaStream_t st, const int64_t* boxes, A... a) {
  // nrep is argument 12 after boxes (see lattice_pot_kernel's parameter list)
  const int nrep = std::get<12>(std::make_tuple(a...));
  static_assert(std::is_same<typename std::tuple_element<12, std::tuple<A...>>::type, int>::value,
                "launch_lattice: argument 12 must be nrep");
  if (nrep <= 2 * kLatBT) lattice_pot_kernel<ND, 2, DM><<<grid, kLatBT, 0, st>>>(boxes, a...);
  else if (nrep <= 3 * kLatBT) lattice_pot_kernel<ND, 3, DM><<<grid, kLatBT, 0, st>>>(boxes, a...);
  else if (nrep <= 4 * kLatBT) lattice_pot_kernel<ND, 4, DM><<<grid, kLatBT, 0, st>>>(boxes, a...);
  else lattice_pot_kernel<ND, 6, DM><<<grid, kLatBT, 0, st>>>(boxes, a...);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

template <int ND, class... A>
int launch_lattice(unsigned grid, cudaStream_t st, const int64_t* boxes, A... a) {
  if (grid == 0) return LB_OK;
  // the dipole mask of the chunk's densities is argument 10 after boxes
  static_assert(std::is_same<typename std::tuple_element<10, std::tuple<A...>>::type, int>::value,
                "launch_lattice: argument 10 must be the dipole mask");
  const unsigned dm = (unsigned)std::get<10>(std::make_tuple(a...)) & ((1u << ND) - 1u);
  constexpr unsigned ALL = (1u << ND) - 1u;
  if (dm == 0u) return launch_lattice_dm<ND, 0u>(grid, st, boxes, a...);
  if constexpr (ND == 2) {
    if (dm == 1u) return launch_lattice_dm<ND, 1u>(grid, st, boxes, a...);
    if (dm == 2u) return launch_lattice_dm<ND, 2u>(grid, st, boxes, a...);
  }
  return launch_lattice_dm<ND, ALL>(grid, st, boxes, a...);
}

// ---------------------------------------------------------------------------
// Chebyshev-grid representation kernels (fmm.py:389-533)

// Lagrange basis at Chebyshev nodes: L = T @ vinv, with derivatives
// (fmm.py:393-428); n <= 16
__device__ void lag_basis(int n, const double* __restrict__ vinv, double x, double* L, double* dL,
                          double* d2L, int nderiv) {
  double t[16], dt[16], d2t[16];
  t[0] = 1.0; dt[0] = 0.0; d2t[0] = 0.0;
  if (n > 1) { t[1] = x; dt[1] = 1.0; d2t[1] = 0.0; }
  for (int k = 2; k < n; ++k) {
    t[k] = 2.0 * x * t[k - 1] - t[k - 2];
    dt[k] = 2.0 * t[k - 1] + 2.0 * x * dt[k - 1] - dt[k - 2];
    d2t[k] = 4.0 * dt[k - 1] + 2.0 * x * d2t[k - 1] - d2t[k - 2];
  }
  for (int a = 0; a < n; ++a) {
    double s0 = 0.0, s1 = 0.0, s2 = 0.0;
    for (int k = 0; k < n; ++k) {
      const double v = vinv[k * n + a];
      s0 += t[k] * v;
      if (nderiv >= 1) s1 += dt[k] * v;
      if (nderiv >= 2) s2 += d2t[k] * v;
    }
    L[a] = s0;
    if (nderiv >= 1) dL[a] = s1;
    if (nderiv >= 2) d2L[a] = s2;
  }
}

// P2M grid anterpolation (fmm.py:484-504): one block per source leaf,
// W[(a*n+b)*n+c, l] = sum_j Lx Ly Lz q + (1/h) (dLx Ly Lz vx + ...)
template <int ND>
__global__ void __launch_bounds__(256) p2m_grid_kernel(
    const int64_t* __restrict__ leaves, const double* __restrict__ bctr,
    const double* __restrict__ bhalf, const int64_t* __restrict__ bsrc,
    const double* __restrict__ spos, const double* __restrict__ cs, const double* __restrict__ vs,
    int64_t ns, int hd, int n, const double* __restrict__ vinv, double* __restrict__ up) {
  constexpr int TJ = 16;
  __shared__ double Ls[TJ][3][16], dLs[TJ][3][16];
  __shared__ double q[TJ][ND], v[TJ][ND][3];
  const int64_t b = leaves[blockIdx.x];
  const double h = bhalf[b], ih = 1.0 / h;
  const double c[3] = {bctr[3 * b], bctr[3 * b + 1], bctr[3 * b + 2]};
  const int64_t s0 = bsrc[2 * b], s1 = bsrc[2 * b + 1];
  const int nrep = n * n * n;
  for (int o0 = 0; o0 < nrep; o0 += blockDim.x) {
    const int o = o0 + threadIdx.x;
    const int ia = o / (n * n), ib = (o / n) % n, ic = o % n;
    double acc[ND];
#pragma unroll
    for (int l = 0; l < ND; ++l) acc[l] = 0.0;
    for (int64_t j0 = s0; j0 < s1; j0 += TJ) {
      const int nj = (int)min((int64_t)TJ, s1 - j0);
      __syncthreads();
      if (threadIdx.x < nj * 3) {
        const int jj = threadIdx.x / 3, ax = threadIdx.x % 3;
        const double tloc = (spos[3 * (j0 + jj) + ax] - c[ax]) / h;  // fmm.py:832
        double d2[16];
        lag_basis(n, vinv, tloc, Ls[jj][ax], dLs[jj][ax], d2, hd ? 1 : 0);
      }
      if (threadIdx.x < nj * ND) {
        const int jj = threadIdx.x / ND, l = threadIdx.x % ND;
        q[jj][l] = cs[(int64_t)l * ns + j0 + jj];
        for (int k = 0; k < 3; ++k) v[jj][l][k] = hd ? vs[((int64_t)l * ns + j0 + jj) * 3 + k] : 0.0;
      }
      __syncthreads();
      if (o < nrep) {
        for (int jj = 0; jj < nj; ++jj) {
          const double lx = Ls[jj][0][ia], ly = Ls[jj][1][ib], lz = Ls[jj][2][ic];
          const double w = lx * ly * lz;
#pragma unroll
          for (int l = 0; l < ND; ++l) {
            acc[l] = fma(w, q[jj][l], acc[l]);
            if (hd) {
              const double g = dLs[jj][0][ia] * ly * lz * v[jj][l][0] +
                               lx * dLs[jj][1][ib] * lz * v[jj][l][1] +
                               lx * ly * dLs[jj][2][ic] * v[jj][l][2];
              acc[l] = fma(ih, g, acc[l]);
            }
          }
        }
      }
    }
    if (o < nrep) {
#pragma unroll
      for (int l = 0; l < ND; ++l) up[(b * ND + l) * (int64_t)nrep + o] = acc[l];
    }
  }
}

// separable 3 x 1-D transform of one n^3 block (per (child,parent) pair):
//   mode 0 (M2M, fmm.py:866-868): dst_p[a,b,c] += sum_def F0[d,a] F1[e,b] F2[f,c] src_c[d,e,f]
//   mode 1 (L2L, fmm.py:930-932): dst_c[d,e,f] += sum_abc F0[d,a] F1[e,b] F2[f,c] src_p[a,b,c]
// F_k = m2m_1d[octant bit k] (n x n: child node x parent basis)
template <int ND>
__global__ void __launch_bounds__(256) grid_tensor_kernel(const int64_t* __restrict__ child,
                                                          const int64_t* __restrict__ parent,
                                                          const int64_t* __restrict__ octant_of,
                                                          const double* __restrict__ f1d, int n,
                                                          const double* __restrict__ src,
                                                          double* __restrict__ dst, int mode) {
  extern __shared__ double sm[];
  const int n3 = n * n * n;
  double* A = sm;        // n^3
  double* B = sm + n3;   // n^3
  const int64_t c = child[blockIdx.x], p = parent[blockIdx.x];
  const int oct = (int)octant_of[c];
  const double* F[3] = {f1d + (oct & 1) * n * n, f1d + ((oct >> 1) & 1) * n * n,
                        f1d + ((oct >> 2) & 1) * n * n};
  const int64_t sbox = mode == 0 ? c : p, dbox = mode == 0 ? p : c;
  for (int l = 0; l < ND; ++l) {
    const double* s = src + (sbox * ND + l) * (int64_t)n3;
    __syncthreads();
    for (int o = threadIdx.x; o < n3; o += blockDim.x) A[o] = s[o];
    __syncthreads();
    // contract axis 2, then 1, then 0; M(u,v) = F[u*n+v] (row = child node)
    for (int o = threadIdx.x; o < n3; o += blockDim.x) {  // B[i,j,z] over A[i,j,k]
      const int i = o / (n * n), j = (o / n) % n, z = o % n;
      double acc = 0.0;
      for (int k = 0; k < n; ++k)
        acc += (mode == 0 ? F[2][k * n + z] : F[2][z * n + k]) * A[(i * n + j) * n + k];
      B[o] = acc;
    }
    __syncthreads();
    for (int o = threadIdx.x; o < n3; o += blockDim.x) {  // A[i,y,z] over B[i,j,z]
      const int i = o / (n * n), y = (o / n) % n, z = o % n;
      double acc = 0.0;
      for (int j = 0; j < n; ++j)
        acc += (mode == 0 ? F[1][j * n + y] : F[1][y * n + j]) * B[(i * n + j) * n + z];
      A[o] = acc;
    }
    __syncthreads();
    double* d = dst + (dbox * ND + l) * (int64_t)n3;
    for (int o = threadIdx.x; o < n3; o += blockDim.x) {  // out[x,y,z] over A[i,y,z]
      const int x = o / (n * n), yz = o % (n * n);
      double acc = 0.0;
      for (int i = 0; i < n; ++i)
        acc += (mode == 0 ? F[0][i * n + x] : F[0][x * n + i]) * A[i * n * n + yz];
      d[o] += acc;
    }
  }
}

// ---------------------------------------------------------------------------
// M2L staging

// sources outside the owned range zeroed (the P2M input of a rank's upward pass)
__global__ void mask_sources_kernel(const double* __restrict__ cs, const double* __restrict__ vs,
                                    const uint8_t* __restrict__ own, int64_t ns, int nd,
                                    double* __restrict__ cs_own, double* __restrict__ vs_own) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= ns) return;
  const double m = own[p] ? 1.0 : 0.0;
  for (int l = 0; l < nd; ++l) {
    cs_own[(int64_t)l * ns + p] = m * cs[(int64_t)l * ns + p];
    for (int k = 0; k < 3; ++k) vs_own[((int64_t)l * ns + p) * 3 + k] = m * vs[((int64_t)l * ns + p) * 3 + k];
  }
}

// surface M2M, second half: up[parent, l] += sum over its children (octant
// order, fmm.py:853-871) of the staged m2m[octant] @ up[child, l]
__global__ void m2m_sum_kernel(const double* __restrict__ Y, const int64_t* __restrict__ child8,
                               const int64_t* __restrict__ parents, int64_t np, int nd, int nrep,
                               double* __restrict__ up) {
  const int64_t pl = blockIdx.x;
  if (pl >= np * nd) return;
  const int64_t p = pl / nd;
  const int l = (int)(pl % nd);
  const int64_t* ch = child8 + 8 * p;
  double* u = up + (parents[p] * nd + l) * (int64_t)nrep;
  for (int i = threadIdx.x; i < nrep; i += blockDim.x) {
    double acc = u[i];
#pragma unroll
    for (int o = 0; o < 8; ++o)
      if (ch[o] >= 0) acc += Y[(ch[o] * nd + l) * (int64_t)nrep + i];
    u[i] = acc;
  }
}

// per unique target t of the chunk: dc[t,l,i] += sum over its pairs (fixed
// order) of Y[(pi-p0)*nd+l, perm[off(pi), i]]
__global__ void m2l_accum_kernel(const double* __restrict__ Y, const int64_t* __restrict__ vtgts,
                                 const int64_t* __restrict__ tpair_off, const int32_t* __restrict__ voff,
                                 const int32_t* __restrict__ perm, int64_t t0, int64_t p0, int nd,
                                 int nrep, double* __restrict__ dc) {
  const int64_t ti = t0 + blockIdx.x;
  const int64_t tb = vtgts[ti];
  const int64_t pb = tpair_off[ti], pe = tpair_off[ti + 1];
  for (int l = 0; l < nd; ++l) {
    double* d = dc + (tb * nd + l) * (int64_t)nrep;
    for (int i = threadIdx.x; i < nrep; i += blockDim.x) {
      double acc = 0.0;
      for (int64_t pi = pb; pi < pe; ++pi)
        acc += Y[((pi - p0) * nd + l) * (int64_t)nrep + perm[(int64_t)voff[pi] * nrep + i]];
      d[i] += acc;
    }
  }
}

// ---------------------------------------------------------------------------
// leaf stage

// grid L2T (fmm.py:507-533): tout[l, t, comp] += interpolant of local[b].
// One block per target leaf, one thread per target; the leaf's local
// coefficients (n^3) and every thread's 1-D bases (value / d / d2 per axis)
// live in shared memory, the contraction runs z -> y -> x.
constexpr int kL2tBT = 64;

template <int ND>
__global__ void __launch_bounds__(kL2tBT) l2t_grid_kernel(
    const int64_t* __restrict__ leaves, const double* __restrict__ bctr,
    const double* __restrict__ bhalf, const int64_t* __restrict__ btgt,
    const double* __restrict__ tpos, int64_t nt, int n, const double* __restrict__ vinv,
    const double* __restrict__ loc, int level, double* __restrict__ tout) {
  extern __shared__ double sm[];
  const int n3 = n * n * n;
  const int nb = 3 * (level + 1) * n;  // bases per thread
  double* W = sm;                       // n^3
  double* Bs = sm + n3;                 // kL2tBT * nb
  const int64_t b = leaves[blockIdx.x];
  const double h = bhalf[b], ih = 1.0 / h;
  const double c[3] = {bctr[3 * b], bctr[3 * b + 1], bctr[3 * b + 2]};
  const int64_t t0 = btgt[2 * b], t1 = btgt[2 * b + 1];
  double* B = Bs + threadIdx.x * nb;  // [axis][deriv][node]
  for (int64_t tb = t0; tb < t1; tb += kL2tBT) {
    const int64_t t = tb + threadIdx.x;
    const bool in = t < t1;
    if (in) {
      for (int ax = 0; ax < 3; ++ax) {
        double* Lax = B + ax * (level + 1) * n;
        lag_basis(n, vinv, (tpos[3 * t + ax] - c[ax]) / h, Lax, Lax + n, Lax + 2 * n, level);
      }
    }
    const double* X0 = B;
    const double* Y0 = B + (level + 1) * n;
    const double* Z0 = B + 2 * (level + 1) * n;
    for (int l = 0; l < ND; ++l) {
      __syncthreads();
      const double* w = loc + (b * ND + l) * (int64_t)n3;
      for (int o = threadIdx.x; o < n3; o += kL2tBT) W[o] = w[o];
      __syncthreads();
      if (!in) continue;
      double r[10] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0};
      for (int ia = 0; ia < n; ++ia) {
        double s00 = 0, s01 = 0, s10 = 0, s02 = 0, s11 = 0, s20 = 0;
        for (int ib = 0; ib < n; ++ib) {
          double z0 = 0, z1 = 0, z2 = 0;
          const double* wr = W + (ia * n + ib) * n;
          for (int ic = 0; ic < n; ++ic) {
            const double wv = wr[ic];
            z0 = fma(Z0[ic], wv, z0);
            if (level >= 1) z1 = fma(Z0[n + ic], wv, z1);
            if (level >= 2) z2 = fma(Z0[2 * n + ic], wv, z2);
          }
          const double y0 = Y0[ib];
          s00 = fma(y0, z0, s00);
          if (level >= 1) {
            const double y1 = Y0[n + ib];
            s01 = fma(y0, z1, s01);
            s10 = fma(y1, z0, s10);
            if (level >= 2) {
              s02 = fma(y0, z2, s02);
              s11 = fma(y1, z1, s11);
              s20 = fma(Y0[2 * n + ib], z0, s20);
            }
          }
        }
        const double x0 = X0[ia];
        r[0] = fma(x0, s00, r[0]);
        if (level >= 1) {
          const double x1 = X0[n + ia];
          r[1] = fma(x1, s00, r[1]);  // d/dx
          r[2] = fma(x0, s10, r[2]);  // d/dy
          r[3] = fma(x0, s01, r[3]);  // d/dz
          if (level >= 2) {
            r[4] = fma(X0[2 * n + ia], s00, r[4]);  // xx
            r[5] = fma(x0, s20, r[5]);              // yy
            r[6] = fma(x0, s02, r[6]);              // zz
            r[7] = fma(x1, s10, r[7]);              // xy
            r[8] = fma(x1, s01, r[8]);              // xz
            r[9] = fma(x0, s11, r[9]);              // yz
          }
        }
      }
      double* o = tout + ((int64_t)l * nt + t) * 10;
      o[0] += r[0];
      if (level >= 1)
        for (int k = 1; k < 4; ++k) o[k] += ih * r[k];
      if (level >= 2)
        for (int k = 4; k < 10; ++k) o[k] += ih * ih * r[k];
    }
  }
}

inline size_t l2t_smem(int n, int level) {
  return sizeof(double) * ((size_t)n * n * n + (size_t)kL2tBT * 3 * (level + 1) * n);
}

// Fused leaf P2P (fmm.py:947-988).  The source sets of a target leaf -- its
// U-list leaves (real charges/dipoles), its own downward-equivalent charges
// (surface) and its W-list boxes' upward-equivalent charges -- are walked as
// ONE virtual list so every shared-memory tile is full; the block's threads
// are split into kSplit source phases per target and combined at the end.
#ifndef LB_LEAF_BT
#define LB_LEAF_BT 128
#endif
constexpr int kLeafBT = LB_LEAF_BT;
constexpr int kLeafTS = 256;
constexpr int kLeafMaxSets = 512;

// Projected pair of the two-density A3 call (fmm_apply_a3proj), where density
// X = charge c0 with dipole -c1 n_s and density B = charge c1.  Record
// [x y z | cX  n_s | cB  0]: real sources carry their normal n_s in X's
// dipole slots (their X dipole is -cB n_s by construction), equivalent
// sources zeros.  Outputs per target:
//   a[0] += -n.grad X + n.H_B.n = r^-3 [cX (n.r) + cB Kspp],
//           Kspp = 3 (n.r)(dn.r)/r^2 - n.dn, dn = n - n_s  (formed first: the
//           accurate form of FarA3c; n_s = 0 gives the equivalent sources'
//           charge-only terms exactly)
//   a[1] += cB / r          a[2] += n.grad B = -cB (n.r) / r^3
// ~40 flop instead of the ~130 of two densities' gradients and Hessians.
__device__ __forceinline__ void pair_a3(double tx, double ty, double tz, double nx, double ny,
                                        double nz, const double* __restrict__ rec, double* a) {
  const double r0 = tx - rec[0], r1 = ty - rec[1], r2 = tz - rec[2];
  const double rr = fma(r2, r2, fma(r1, r1, r0 * r0));
  const double invr = inv_sqrt_skip(rr);
  const double invr2 = invr * invr;
  const double invr3 = invr * invr2;
  const double rnt = fma(nz, r2, fma(ny, r1, nx * r0));
  const double dn0 = nx - rec[4], dn1 = ny - rec[5], dn2 = nz - rec[6];
  const double rdn = fma(dn2, r2, fma(dn1, r1, dn0 * r0));
  const double ndn = fma(nz, dn2, fma(ny, dn1, nx * dn0));
  const double cX = rec[3], cB = rec[7];
  const double kspp = fma(3.0 * rnt * rdn, invr2, -ndn);
  a[0] = fma(invr3, fma(cX, rnt, cB * kspp), a[0]);
  a[1] = fma(cB, invr, a[1]);
  a[2] = fma(-cB * invr3, rnt, a[2]);
}

template <int ND, bool HD, int LEVEL, bool A3P = false>
__global__ void __launch_bounds__(kLeafBT) leaf_kernel(
    const int64_t* __restrict__ order, const int64_t* __restrict__ items, double* __restrict__ part,
    const int64_t* __restrict__ leaves, const int64_t* __restrict__ u_off,
    const int64_t* __restrict__ u_list, const int64_t* __restrict__ w_off,
    const int64_t* __restrict__ w_list, const double* __restrict__ bctr,
    const double* __restrict__ bhalf, const int64_t* __restrict__ bsrc,
    const int64_t* __restrict__ btgt, const double* __restrict__ spos,
    const double* __restrict__ tpos, const double* __restrict__ cs, const double* __restrict__ vs,
    int64_t ns, int64_t nt, const double* __restrict__ pts, int nrep, int surface, double de_scale,
    double ue_scale, const double* __restrict__ loc, const double* __restrict__ up,
    double* __restrict__ tout, const double* __restrict__ tnrm = nullptr,
    const double* __restrict__ snrm = nullptr) {
  using Lay = SrcLayout<ND, true, HD>;
  constexpr int S = Lay::stride;
  constexpr int NC = ncomp(LEVEL);
  constexpr int NA = A3P ? 3 : ND * NC;
  static_assert(!A3P || (ND == 2 && HD), "projected leaf: the two-density A3 call only");
  constexpr int kTS = S > 8 ? kLeafTS / 2 : kLeafTS;
  __shared__ __align__(16) double sh[kTS * S];
  __shared__ int64_t set_end[kLeafMaxSets + 1];
  __shared__ int64_t set_box[kLeafMaxSets];
  __shared__ double red[kLeafBT];
  // work item: target leaf li, virtual sources [vb, ve), partial slot (or -1)
  const int64_t it = order[blockIdx.x];
  const int64_t li = items[4 * it], vb = items[4 * it + 1];
  const int64_t ve = items[4 * it + 2], poff = items[4 * it + 3];
  const int64_t b = leaves[li];
  const int64_t t0 = btgt[2 * b], t1 = btgt[2 * b + 1];
  // leaves hold few targets (~17 on average at ncrit 120): the target pass
  // is the leaf's own size (not a power of two: 17 targets would leave 15 of
  // every 32 threads idle) and the remaining threads take other source phases
  // A leaf whose target count is not close to a divisor of the block (ncrit
  // 300 on a 4x oversampled surface: ~75 of 128; a 150-target leaf: 128 + 22)
  // would leave many threads idle: cut its targets into P balanced passes of
  // ceil(nt / P) so that kSplit = kLeafBT / kTgt source phases fill the
  // block; P minimises passes x sources-per-phase (+5% per pass for the
  // re-staged tiles)
  const int ntl = (int)max((int64_t)1, t1 - t0);
  int kTgt = min(ntl, kLeafBT);
  {
    double best = 1e30;
    for (int p = (ntl + kLeafBT - 1) / kLeafBT; p <= 16; ++p) {
      const int kt = (ntl + p - 1) / p;
      const double cost = p * (1.0 / (kLeafBT / kt) + 0.05);
      if (cost < best - 1e-12) {
        best = cost;
        kTgt = kt;
      }
      if (kt == 1) break;
    }
  }
  const int kSplit = kLeafBT / kTgt;
  const int64_t ub = u_off[li], nu = u_off[li + 1] - ub;
  const int64_t wb = w_off[li], nw = w_off[li + 1] - wb;
  const int64_t nde = surface ? 1 : 0;
  const int64_t nsets_all = nu + nde + nw;
  const int ti = threadIdx.x % kTgt, ph = threadIdx.x / kTgt;
  const bool active = ph < kSplit;  // the last kLeafBT % kTgt threads only stage sources
  for (int64_t tb = t0; tb < t1; tb += kTgt) {
    const int64_t t = tb + ti;
    const bool in = active && t < t1;
    const double tx = in ? tpos[3 * t] : 0.0, ty = in ? tpos[3 * t + 1] : 0.0,
                 tz = in ? tpos[3 * t + 2] : 0.0;
    double nx = 0.0, ny = 0.0, nz = 0.0;
    if (A3P && in) {
      nx = tnrm[3 * t];
      ny = tnrm[3 * t + 1];
      nz = tnrm[3 * t + 2];
    }
    double acc[NA];
#pragma unroll
    for (int a = 0; a < NA; ++a) acc[a] = 0.0;
    int64_t vbase = 0;  // virtual index of this batch's first source
    for (int64_t sb0 = 0; sb0 < nsets_all && vbase < ve; sb0 += kLeafMaxSets) {
      const int nsets = (int)min((int64_t)kLeafMaxSets, nsets_all - sb0);
      // prefix sizes of this batch of source sets: every thread looks its
      // sets up (the list entry and its box's source range are two dependent
      // global loads: one thread walking ~50 sets serially stalled the whole
      // block), then warp 0 scans the counts.  One batch covers the whole
      // list in all but the largest leaves, and it is the same for every
      // target pass: built once then.
      if (sb0 > 0 || nsets_all > kLeafMaxSets || tb == t0) {
        __syncthreads();
        for (int q = threadIdx.x; q < nsets; q += kLeafBT) {
          const int64_t g = sb0 + q;
          int64_t box, cnt;
          if (g < nu) {
            box = u_list[ub + g];
            cnt = bsrc[2 * box + 1] - bsrc[2 * box];
          } else if (g < nu + nde) {
            box = -1 - b;  // own DE set
            cnt = nrep;
          } else {
            box = -1 - w_list[wb + (g - nu - nde)];
            cnt = nrep;
          }
          set_box[q] = box;
          set_end[q] = cnt;
        }
        __syncthreads();
        if (threadIdx.x < 32) {
          int64_t carry = 0;
          for (int q0 = 0; q0 < nsets; q0 += 32) {
            const int q = q0 + threadIdx.x;
            int64_t v = q < nsets ? set_end[q] : 0;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
              const int64_t up = __shfl_up_sync(0xffffffffu, v, o);
              if ((int)threadIdx.x >= o) v += up;
            }
            if (q < nsets) set_end[q] = carry + v;
            carry += __shfl_sync(0xffffffffu, v, 31);
          }
        }
      }
      __syncthreads();
      const int64_t total = set_end[nsets - 1];
      const int64_t vlo = max((int64_t)0, vb - vbase), vhi = min(total, ve - vbase);
      for (int64_t v0 = vlo; v0 < vhi; v0 += kTS) {
        const int n = (int)min((int64_t)kTS, vhi - v0);
        __syncthreads();
        for (int k = threadIdx.x; k < n; k += kLeafBT) {
          const int64_t v = v0 + k;
          int lo = 0, hi = nsets - 1;  // first set with set_end > v
          while (lo < hi) {
            const int mid = (lo + hi) >> 1;
            if (set_end[mid] > v) hi = mid; else lo = mid + 1;
          }
          const int64_t off = v - (lo ? set_end[lo - 1] : 0);
          const int64_t box = set_box[lo];
          double* r = sh + k * S;
          int o = 3;
          if (box >= 0) {  // real sources of a U-list leaf
            const int64_t j = bsrc[2 * box] + off;
            r[0] = spos[3 * j]; r[1] = spos[3 * j + 1]; r[2] = spos[3 * j + 2];
#pragma unroll
            for (int l = 0; l < ND; ++l) {
              r[o++] = cs[(int64_t)l * ns + j];
              if (HD)
                for (int kk = 0; kk < 3; ++kk) r[o++] = vs[((int64_t)l * ns + j) * 3 + kk];
            }
            if (A3P) {  // X's dipole slots carry the source normal (see pair_a3)
              r[4] = snrm[3 * j];
              r[5] = snrm[3 * j + 1];
              r[6] = snrm[3 * j + 2];
            }
          } else {  // equivalent charges: own DE set (loc) or a W box (up)
            const int64_t eb = -1 - box;
            const bool de = eb == b && surface && (lo + sb0) == nu;
            const double fac = de ? de_scale : ue_scale;
            const double* eq = de ? loc : up;
            const double h = bhalf[eb];
            r[0] = bctr[3 * eb] + fac * h * pts[3 * off];
            r[1] = bctr[3 * eb + 1] + fac * h * pts[3 * off + 1];
            r[2] = bctr[3 * eb + 2] + fac * h * pts[3 * off + 2];
#pragma unroll
            for (int l = 0; l < ND; ++l) {
              r[o++] = eq[(eb * ND + l) * (int64_t)nrep + off];
              if (HD)
                for (int kk = 0; kk < 3; ++kk) r[o++] = 0.0;
            }
          }
        }
        __syncthreads();
        // unrolled over sources: independent pair chains give the FP64 pipe
        // ILP (one pair at a time is a serial DADD-DFMA-MUFU-DFMA chain)
        if (active) {
          if constexpr (A3P) {
#pragma unroll 4
            for (int k = ph; k < n; k += kSplit) pair_a3(tx, ty, tz, nx, ny, nz, sh + k * S, acc);
          } else {
#pragma unroll 4
            for (int k = ph; k < n; k += kSplit) pair_generic<ND, true, HD, LEVEL>(tx, ty, tz, sh + k * S, acc);
          }
        }
      }
      vbase += total;
    }
    // combine the source phases (fixed order), one component at a time
    if (kSplit > 1) {
#pragma unroll
      for (int a = 0; a < NA; ++a) {
        __syncthreads();
        red[threadIdx.x] = acc[a];
        __syncthreads();
        if (ph == 0)
          for (int q = 1; q < kSplit; ++q) acc[a] += red[q * kTgt + ti];
      }
    }
    if (in && ph == 0 && poff >= 0) {  // split leaf: this item's partial (reduced in order later)
#pragma unroll
      for (int a = 0; a < NA; ++a) part[poff + (t - t0) * NA + a] = acc[a];
    } else if (in && ph == 0) {
      if constexpr (A3P) {
#pragma unroll
        for (int c = 0; c < 3; ++c) tout[t * 3 + c] = acc[c];
      } else {
#pragma unroll
        for (int l = 0; l < ND; ++l) {
          double* o = tout + ((int64_t)l * nt + t) * 10;
#pragma unroll
          for (int c = 0; c < NC; ++c) o[c] += acc[l * NC + c];
        }
      }
    }
  }
}

// items[4i+3] = slot[i] * width (doubles) for split items, -1 otherwise
__global__ void scale_item_offsets_kernel(int64_t* __restrict__ items, const int64_t* __restrict__ slot,
                                          int64_t n, int64_t width) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) items[4 * i + 3] = slot[i] < 0 ? -1 : slot[i] * width;
}

// partials of split leaves, summed in item order (deterministic) into the
// leaf's outputs: generic acc[l * NC + c] -> tout[(l * nt + t) * 10 + c] (+=,
// the grid L2T is already there); projected acc[a] -> tproj[t * 3 + a]
template <int ND, int NC, bool A3P>
__global__ void leaf_reduce_kernel(const int64_t* __restrict__ split_leaf, const int64_t* __restrict__ item_off,
                                   const int64_t* __restrict__ items, const int64_t* __restrict__ leaves,
                                   const int64_t* __restrict__ btgt, const double* __restrict__ part,
                                   int64_t nt, double* __restrict__ tout) {
  constexpr int NA = A3P ? 3 : ND * NC;
  const int64_t si = blockIdx.x;
  const int64_t li = split_leaf[si];
  const int64_t b = leaves[li];
  const int64_t t0 = btgt[2 * b], t1 = btgt[2 * b + 1];
  const int64_t i0 = item_off[2 * si], i1 = item_off[2 * si + 1];
  for (int64_t x = threadIdx.x; x < (t1 - t0) * NA; x += blockDim.x) {
    const int64_t lt = x / NA;
    const int a = (int)(x - lt * NA);
    double v = 0.0;
    for (int64_t it = i0; it < i1; ++it) v += part[items[4 * it + 3] + x];
    const int64_t t = t0 + lt;
    if (A3P) {
      tout[t * 3 + a] = v;
    } else {
      const int l = a / NC, c = a - l * NC;
      tout[((int64_t)l * nt + t) * 10 + c] += v;
    }
  }
}

// sorted targets -> reference layout
__global__ void fmm_scatter_kernel(const double* __restrict__ tout, const int64_t* __restrict__ tgt_sorted,
                                   int64_t nt, int nd, int d0, int level, double* __restrict__ pot,
                                   double* __restrict__ grad, double* __restrict__ hess) {
  const int64_t idx = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (int64_t)nd * nt) return;
  const int l = (int)(idx / nt);
  const int64_t t = idx - (int64_t)l * nt;
  const double* v = tout + idx * 10;
  const int64_t row = (int64_t)(d0 + l) * nt + tgt_sorted[t];
  pot[row] = v[0];
  if (level >= 1)
    for (int k = 0; k < 3; ++k) grad[row * 3 + k] = v[1 + k];
  if (level >= 2) {
    const double hv[9] = {v[4], v[7], v[8], v[7], v[5], v[9], v[8], v[9], v[6]};
    for (int k = 0; k < 9; ++k) hess[row * 9 + k] = hv[k];
  }
}

// reference-order rows -> sorted rows (target normals) and back (projections)
__global__ void gather_rows3_kernel(const double* __restrict__ in, const int64_t* __restrict__ sorted,
                                    int64_t n, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t r = sorted[t];
  for (int k = 0; k < 3; ++k) out[3 * t + k] = in[3 * r + k];
}
__global__ void scatter_proj_kernel(const double* __restrict__ tproj, const int64_t* __restrict__ sorted,
                                    int64_t n, double* __restrict__ out) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const int64_t r = sorted[t];
  for (int c = 0; c < 3; ++c) out[(int64_t)c * n + r] = tproj[3 * t + c];
}

// ---------------------------------------------------------------------------
// M2L pair grouping on the device (from the device tree build's V list):
// pairs laid out in (target slot, V order), stable radix sort by canonical
// key, then per-(key, target) groups -- the same arrays build_device's host
// path produces.

__global__ void gather3_kernel(const double* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                               double* __restrict__ dst) {
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= n) return;
  const int64_t o = idx[p];
  dst[3 * p] = src[3 * o];
  dst[3 * p + 1] = src[3 * o + 1];
  dst[3 * p + 2] = src[3 * o + 2];
}

__global__ void m2l_count_kernel(const int64_t* __restrict__ id_of, const uint8_t* __restrict__ owned_id,
                                 const int64_t* __restrict__ voff, int64_t nslot, int64_t* __restrict__ cnt) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslot) return;
  const int64_t b = id_of[s];
  cnt[s] = owned_id[b] ? voff[b + 1] - voff[b] : 0;
}

constexpr int kOffR = 8, kOffW = 2 * kOffR + 1;  // dense lattice-offset table

__global__ void m2l_fill_kernel(const int64_t* __restrict__ id_of, const uint8_t* __restrict__ owned_id,
                                const int64_t* __restrict__ voff, const int64_t* __restrict__ vidx,
                                const int64_t* __restrict__ poff, const int64_t* __restrict__ ijk,
                                const int32_t* __restrict__ level, const double* __restrict__ inv_h,
                                const int32_t* __restrict__ off_table, const int32_t* __restrict__ off_key,
                                const int64_t* __restrict__ slot_of, int64_t nslot, int32_t* __restrict__ keys,
                                int64_t* __restrict__ ids, int64_t* __restrict__ tgt, int64_t* __restrict__ src,
                                int32_t* __restrict__ off, double* __restrict__ scale, int* __restrict__ bad) {
  const int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= nslot) return;
  const int64_t b = id_of[s];
  if (!owned_id[b]) return;
  int64_t at = poff[s];
  const double sc = inv_h[level[b]];
  for (int64_t q = voff[b]; q < voff[b + 1]; ++q, ++at) {
    const int64_t c = vidx[q];
    const int64_t dx = ijk[3 * c] - ijk[3 * b], dy = ijk[3 * c + 1] - ijk[3 * b + 1],
                  dz = ijk[3 * c + 2] - ijk[3 * b + 2];
    int d = -1;
    if (llabs(dx) <= kOffR && llabs(dy) <= kOffR && llabs(dz) <= kOffR)
      d = off_table[((dx + kOffR) * kOffW + (dy + kOffR)) * kOffW + (dz + kOffR)];
    if (d < 0) {
      atomicExch(bad, 1);
      d = 0;
    }
    keys[at] = off_key[d];
    ids[at] = at;
    tgt[at] = s;
    src[at] = slot_of[c];
    off[at] = d;
    scale[at] = sc;
  }
}

__global__ void m2l_gather_pairs_kernel(const int64_t* __restrict__ perm, const int32_t* __restrict__ keys_s,
                                        const int64_t* __restrict__ tgt, const int64_t* __restrict__ src,
                                        const int32_t* __restrict__ off, const double* __restrict__ scale,
                                        int64_t n, int64_t* __restrict__ tgt_s, int64_t* __restrict__ src_s,
                                        int32_t* __restrict__ off_s, double* __restrict__ scale_s) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int64_t j = perm[i];
  tgt_s[i] = tgt[j];
  src_s[i] = src[j];
  off_s[i] = off[j];
  scale_s[i] = scale[j];
}

__global__ void m2l_group_flags_kernel(const int32_t* __restrict__ keys_s, const int64_t* __restrict__ tgt_s,
                                       int64_t n, int64_t* __restrict__ flag) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  flag[i] = (i == 0 || keys_s[i] != keys_s[i - 1] || tgt_s[i] != tgt_s[i - 1]) ? 1 : 0;
}

__global__ void m2l_groups_kernel(const int32_t* __restrict__ keys_s, const int64_t* __restrict__ tgt_s,
                                  const int64_t* __restrict__ flag, const int64_t* __restrict__ grp_incl,
                                  int64_t n, int64_t* __restrict__ vtgts, int64_t* __restrict__ tpoff,
                                  int64_t* __restrict__ kpair, int64_t* __restrict__ kgrp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flag[i]) return;
  const int64_t g = grp_incl[i] - 1;
  vtgts[g] = tgt_s[i];
  tpoff[g] = i;
  if (i == 0 || keys_s[i] != keys_s[i - 1]) {
    kpair[keys_s[i]] = i;
    kgrp[keys_s[i]] = g;
  }
}

// ---------------------------------------------------------------------------
// host side: device state

namespace {

template <class T>
int upload(T** dst, const std::vector<T>& v) {
  cudaError_t e = cudaMalloc((void**)dst, std::max<size_t>(v.size() * sizeof(T), 16));
  if (e == cudaSuccess && !v.empty()) e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  if (e != cudaSuccess) return fail(LB_ERR_CUDA, std::string("fmm upload: ") + cudaGetErrorString(e));
  return LB_OK;
}

// M2L pairs from the device V list (see the kernels above); fills the same
// FmmDevice arrays as the host path in build_device
int m2l_pairs_device(lb_fmm_plan* P, const std::vector<uint8_t>& own_id, const std::vector<int32_t>& off_table) {
  FmmTree& t = P->tree;
  FmmDevice& D = P->dev;
  const int64_t nb = t.nbox();
  const int nk = P->ncanon;
  std::vector<void*> tmp;
  auto grab = [&](void** p, size_t bytes) -> cudaError_t {
    cudaError_t e = cudaMalloc(p, std::max<size_t>(bytes, 16));
    if (e == cudaSuccess) tmp.push_back(*p);
    return e;
  };
  struct Free {
    std::vector<void*>& v;
    ~Free() { for (void* p : v) cudaFree(p); }
  } free_tmp{tmp};
  std::vector<double> inv_h(t.nlev);
  for (int l = 0; l < t.nlev; ++l) inv_h[l] = 1.0 / (t.half / std::ldexp(1.0, l));  // fmm.py:879
  int64_t *d_idof, *d_slot, *d_ijk, *cnt, *poff;
  uint8_t* d_own;
  int32_t *d_lev, *d_table, *d_key;
  double* d_invh;
  int* d_bad;
  auto up = [&](void** p, const void* src, size_t bytes) -> cudaError_t {
    cudaError_t e = grab(p, bytes);
    if (e == cudaSuccess && bytes) e = cudaMemcpy(*p, src, bytes, cudaMemcpyHostToDevice);
    return e;
  };
  LB_CUDA(up((void**)&d_idof, P->id_of.data(), 8 * nb));
  LB_CUDA(up((void**)&d_slot, P->slot_of.data(), 8 * nb));
  LB_CUDA(up((void**)&d_ijk, t.ijk.data(), 24 * nb));
  LB_CUDA(up((void**)&d_own, own_id.data(), nb));
  LB_CUDA(up((void**)&d_lev, t.level.data(), 4 * nb));
  LB_CUDA(up((void**)&d_table, off_table.data(), 4 * off_table.size()));
  LB_CUDA(up((void**)&d_key, P->off_key.data(), 4 * P->off_key.size()));
  LB_CUDA(up((void**)&d_invh, inv_h.data(), 8 * inv_h.size()));
  LB_CUDA(grab((void**)&d_bad, sizeof(int)));
  LB_CUDA(cudaMemset(d_bad, 0, sizeof(int)));
  LB_CUDA(grab((void**)&cnt, 8 * (nb + 1)));
  LB_CUDA(grab((void**)&poff, 8 * (nb + 1)));
  LB_CUDA(cudaMemset(cnt + nb, 0, 8));
  const unsigned gb = (unsigned)std::max<int64_t>(1, ceil_div(nb, 256));
  m2l_count_kernel<<<gb, 256>>>(d_idof, d_own, P->tdev.v_off, nb, cnt);
  LB_CHECK_LAUNCH();
  size_t sbytes = 0;
  void* stmp = nullptr;
  LB_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, sbytes, cnt, poff, nb + 1));
  LB_CUDA(grab(&stmp, sbytes));
  LB_CUDA(cub::DeviceScan::ExclusiveSum(stmp, sbytes, cnt, poff, nb + 1));
  int64_t np = 0;
  LB_CUDA(cudaMemcpy(&np, poff + nb, 8, cudaMemcpyDeviceToHost));
  int32_t *keys, *keys_s, *off;
  int64_t *ids, *perm, *tgt, *src, *flag, *grp, *kpair, *kgrp;
  double* scale;
  LB_CUDA(grab((void**)&keys, 4 * np));
  LB_CUDA(grab((void**)&keys_s, 4 * np));
  LB_CUDA(grab((void**)&off, 4 * np));
  LB_CUDA(grab((void**)&ids, 8 * np));
  LB_CUDA(grab((void**)&perm, 8 * np));
  LB_CUDA(grab((void**)&tgt, 8 * np));
  LB_CUDA(grab((void**)&src, 8 * np));
  LB_CUDA(grab((void**)&scale, 8 * np));
  m2l_fill_kernel<<<gb, 256>>>(d_idof, d_own, P->tdev.v_off, P->tdev.v_idx, poff, d_ijk, d_lev, d_invh, d_table,
                               d_key, d_slot, nb, keys, ids, tgt, src, off, scale, d_bad);
  LB_CHECK_LAUNCH();
  int bad = 0;
  LB_CUDA(cudaMemcpy(&bad, d_bad, sizeof(int), cudaMemcpyDeviceToHost));
  if (bad) return fail(LB_ERR_ARG, "fmm: V-list offset without an M2L operator");
  int kbits = 1;
  while ((1 << kbits) < nk) ++kbits;
  size_t rbytes = 0;
  void* rtmp = nullptr;
  LB_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, rbytes, keys, keys_s, ids, perm, np, 0, kbits));
  LB_CUDA(grab(&rtmp, rbytes));
  LB_CUDA(cub::DeviceRadixSort::SortPairs(rtmp, rbytes, keys, keys_s, ids, perm, np, 0, kbits));  // stable
  LB_CUDA(cudaMalloc((void**)&D.v_src, std::max<int64_t>(16, 8 * np)));
  LB_CUDA(cudaMalloc((void**)&D.v_off_idx, std::max<int64_t>(16, 4 * np)));
  LB_CUDA(cudaMalloc((void**)&D.v_scale, std::max<int64_t>(16, 8 * np)));
  int64_t* tgt_s = ids;  // reuse
  const unsigned gp = (unsigned)std::max<int64_t>(1, ceil_div(np, 256));
  m2l_gather_pairs_kernel<<<gp, 256>>>(perm, keys_s, tgt, src, off, scale, np, tgt_s, D.v_src, D.v_off_idx,
                                       D.v_scale);
  LB_CHECK_LAUNCH();
  flag = src;  // reuse (gathered already)
  grp = tgt;
  m2l_group_flags_kernel<<<gp, 256>>>(keys_s, tgt_s, np, flag);
  LB_CHECK_LAUNCH();
  size_t ibytes = 0;
  void* itmp = nullptr;
  LB_CUDA(cub::DeviceScan::InclusiveSum(nullptr, ibytes, flag, grp, np));
  LB_CUDA(grab(&itmp, ibytes));
  if (np) LB_CUDA(cub::DeviceScan::InclusiveSum(itmp, ibytes, flag, grp, np));
  int64_t ng = 0;
  if (np) LB_CUDA(cudaMemcpy(&ng, grp + np - 1, 8, cudaMemcpyDeviceToHost));
  LB_CUDA(cudaMalloc((void**)&D.v_tgts, std::max<int64_t>(16, 8 * ng)));
  LB_CUDA(cudaMalloc((void**)&D.v_tgt_pair_off, 8 * (ng + 1)));
  LB_CUDA(grab((void**)&kpair, 8 * std::max(nk, 1)));
  LB_CUDA(grab((void**)&kgrp, 8 * std::max(nk, 1)));
  LB_CUDA(cudaMemset(kpair, 0xff, 8 * std::max(nk, 1)));
  LB_CUDA(cudaMemset(kgrp, 0xff, 8 * std::max(nk, 1)));
  m2l_groups_kernel<<<gp, 256>>>(keys_s, tgt_s, flag, grp, np, D.v_tgts, D.v_tgt_pair_off, kpair, kgrp);
  LB_CHECK_LAUNCH();
  LB_CUDA(cudaMemcpy(D.v_tgt_pair_off + ng, &np, 8, cudaMemcpyHostToDevice));
  D.v_tpoff_host.resize(ng + 1);
  LB_CUDA(cudaMemcpy(D.v_tpoff_host.data(), D.v_tgt_pair_off, 8 * (ng + 1), cudaMemcpyDeviceToHost));
  std::vector<int64_t> kp(nk), kg(nk);
  if (nk) {
    LB_CUDA(cudaMemcpy(kp.data(), kpair, 8 * nk, cudaMemcpyDeviceToHost));
    LB_CUDA(cudaMemcpy(kg.data(), kgrp, 8 * nk, cudaMemcpyDeviceToHost));
  }
  D.v_key_pair_off.assign(nk + 1, np);
  D.v_key_tgt_off.assign(nk + 1, ng);
  for (int k = nk - 1; k >= 0; --k) {  // empty keys start where the next key does
    D.v_key_pair_off[k] = kp[k] >= 0 ? kp[k] : D.v_key_pair_off[k + 1];
    D.v_key_tgt_off[k] = kg[k] >= 0 ? kg[k] : D.v_key_tgt_off[k + 1];
  }
  D.max_key_pairs = 0;
  for (int k = 0; k < nk; ++k)
    D.max_key_pairs = std::max<int64_t>(D.max_key_pairs, D.v_key_pair_off[k + 1] - D.v_key_pair_off[k]);
  return LB_OK;
}

int build_device(lb_fmm_plan* P) {
  const bool verbose = std::getenv("LB_FMM_VERBOSE") != nullptr;
  auto tick = std::chrono::steady_clock::now();
  auto mark = [&](const char* what) {
    const auto now = std::chrono::steady_clock::now();
    if (verbose)
      std::fprintf(stderr, "build_device %-12s %8.1f ms\n", what,
                   std::chrono::duration<double, std::milli>(now - tick).count());
    tick = now;
  };
  FmmTree& t = P->tree;
  FmmDevice& D = P->dev;
  const int64_t nb = t.nbox();
  const int nrep = P->nrep;
  // slots: boxes level by level (ascending id within a level)
  P->slot_of.assign(nb, -1);
  P->id_of.clear();
  std::vector<int64_t> level_slot_off{0};
  for (int l = 0; l < t.nlev; ++l) {
    for (int64_t b : t.levels[l]) {
      P->slot_of[b] = (int64_t)P->id_of.size();
      P->id_of.push_back(b);
    }
    level_slot_off.push_back((int64_t)P->id_of.size());
  }
  const auto& S = P->slot_of;
  // owned targets (lb_fmm_plan_set_target_range): a sharded apply replicates
  // the reference's tree on every rank and runs the downward pass and the
  // leaf stage only where its own targets are; owned(b) counts them below b
  std::vector<int64_t> own_pref(t.nt + 1, 0);
  for (int64_t q = 0; q < t.nt; ++q) {
    const int64_t o = t.tgt_sorted[q];
    const bool mine = P->own_t1 < 0 || (o >= P->own_t0 && o < P->own_t1);
    own_pref[q + 1] = own_pref[q] + (mine ? 1 : 0);
  }
  auto owned = [&](int64_t b) { return own_pref[t.tgt_hi[b]] - own_pref[t.tgt_lo[b]]; };
  std::vector<uint8_t> own_id(nb);
  for (int64_t b = 0; b < nb; ++b) own_id[b] = owned(b) > 0 ? 1 : 0;
  // owned sources (lb_fmm_plan_set_source_range): a rank's upward pass (P2M
  // + M2M) covers only its own sources; the partial expansions are summed
  // across the ranks by the upward hook before the M2L
  const bool src_range = P->own_s1 >= 0;
  std::vector<int64_t> sown_pref(t.ns + 1, 0);
  std::vector<uint8_t> src_own(src_range ? t.ns : 0);
  for (int64_t q = 0; q < t.ns; ++q) {
    const int64_t o = t.src_sorted[q];
    const bool mine = !src_range || (o >= P->own_s0 && o < P->own_s1);
    if (src_range) src_own[q] = mine ? 1 : 0;
    sown_pref[q + 1] = sown_pref[q] + (mine ? 1 : 0);
  }
  auto nsrc_own = [&](int64_t b) { return sown_pref[t.src_hi[b]] - sown_pref[t.src_lo[b]]; };
  const bool dev_tree = P->tdev.spos != nullptr;
  std::vector<double> ctr(3 * nb), hf(nb), spos_s(dev_tree ? 0 : 3 * t.ns), tpos_s(dev_tree ? 0 : 3 * t.nt);
  std::vector<int64_t> bsrc(2 * nb), btgt(2 * nb), octant(nb, 0);
  for (int64_t b = 0; b < nb; ++b) {
    const int64_t s = S[b];
    t.box_center(b, &ctr[3 * s]);
    hf[s] = t.box_half(b);
    bsrc[2 * s] = t.src_lo[b];
    bsrc[2 * s + 1] = t.src_hi[b];
    btgt[2 * s] = t.tgt_lo[b];
    btgt[2 * s + 1] = t.tgt_hi[b];
    if (b > 0) {
      const int64_t p = t.parent[b];
      const int ox = (int)(t.ijk[3 * b] - 2 * t.ijk[3 * p]);
      const int oy = (int)(t.ijk[3 * b + 1] - 2 * t.ijk[3 * p + 1]);
      const int oz = (int)(t.ijk[3 * b + 2] - 2 * t.ijk[3 * p + 2]);
      octant[s] = ox | (oy << 1) | (oz << 2);  // bit k = offset along axis k
    }
  }
  if (dev_tree) {  // positions and sorted index lists are on the device already
    auto dev_copy = [&](int64_t** dst, const int64_t* src, int64_t n) -> cudaError_t {
      cudaError_t e = cudaMalloc((void**)dst, std::max<size_t>(16, 8 * n));
      if (e == cudaSuccess && n) e = cudaMemcpy(*dst, src, 8 * n, cudaMemcpyDeviceToDevice);
      return e;
    };
    LB_CUDA(dev_copy(&D.src_sorted, P->tdev.src_sorted, t.ns));
    LB_CUDA(dev_copy(&D.tgt_sorted, P->tdev.tgt_sorted, t.nt));
    LB_CUDA(cudaMalloc((void**)&D.spos, std::max<size_t>(16, 24 * t.ns)));
    LB_CUDA(cudaMalloc((void**)&D.tpos, std::max<size_t>(16, 24 * t.nt)));
    if (t.ns) {
      gather3_kernel<<<(unsigned)ceil_div(t.ns, 256), 256>>>(P->tdev.spos, D.src_sorted, t.ns, D.spos);
      LB_CHECK_LAUNCH();
    }
    if (t.nt) {
      gather3_kernel<<<(unsigned)ceil_div(t.nt, 256), 256>>>(P->tdev.tpos, D.tgt_sorted, t.nt, D.tpos);
      LB_CHECK_LAUNCH();
    }
    mark("geometry");
  } else {
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < t.ns; ++p)
      for (int k = 0; k < 3; ++k) spos_s[3 * p + k] = P->spos[3 * t.src_sorted[p] + k];
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < t.nt; ++p)
      for (int k = 0; k < 3; ++k) tpos_s[3 * p + k] = P->tpos[3 * t.tgt_sorted[p] + k];
    mark("geometry");
    LB_TRY(upload(&D.spos, spos_s));
    LB_TRY(upload(&D.tpos, tpos_s));
    LB_TRY(upload(&D.src_sorted, t.src_sorted));
    LB_TRY(upload(&D.tgt_sorted, t.tgt_sorted));
  }
  LB_TRY(upload(&D.bctr, ctr));
  LB_TRY(upload(&D.bhalf, hf));
  LB_TRY(upload(&D.bsrc, bsrc));
  LB_TRY(upload(&D.btgt, btgt));
  int64_t* doct = nullptr;
  LB_TRY(upload(&doct, octant));
  D.vinv = nullptr;
  // operators
  LB_TRY(upload(&D.pts, P->pts));
  if (P->rep == 0) {
    LB_TRY(upload(&D.pinv_up, P->pinv_up));
    LB_TRY(upload(&D.pinv_dn, P->pinv_dn));
    LB_TRY(upload(&D.l2l, P->l2l));
    // the 8 child-octant operators in octant order (x | y<<1 | z<<2): the
    // reference lists them by 4*ox + 2*oy + oz (fmm.py:307-317)
    const int64_t nn = (int64_t)nrep * nrep;
    std::vector<double> mo(8 * nn), lo(8 * nn);
    for (int oct = 0; oct < 8; ++oct) {
      const int r = ((oct & 1) << 2) | (oct & 2) | ((oct >> 2) & 1);
      std::copy(P->m2m.begin() + r * nn, P->m2m.begin() + (r + 1) * nn, mo.begin() + oct * nn);
      std::copy(P->l2l.begin() + r * nn, P->l2l.begin() + (r + 1) * nn, lo.begin() + oct * nn);
    }
    LB_TRY(upload(&D.m2m_oct, mo));
    LB_TRY(upload(&D.l2l_oct, lo));
  } else {
    LB_TRY(upload(&D.vinv, P->vinv));
  }
  LB_TRY(upload(&D.m2m, P->m2m));
  LB_TRY(upload(&D.canon, P->canon));
  std::vector<int32_t> pinv(P->off_perm.size());
  for (int d = 0; d < P->noff; ++d)
    for (int i = 0; i < nrep; ++i) pinv[(int64_t)d * nrep + P->off_perm[(int64_t)d * nrep + i]] = i;
  LB_TRY(upload(&D.perm, P->off_perm));
  LB_TRY(upload(&D.perm_inv, pinv));
  mark("uploads");
  // P2M leaves (fmm.py:826) and M2M / L2L groups per (level, octant)
  std::vector<int64_t> p2m;
  for (int64_t b = 0; b < nb; ++b)
    if (t.is_leaf[b] && t.src_hi[b] > t.src_lo[b] && nsrc_own(b) > 0) p2m.push_back(S[b]);
  // heaviest leaves first: one CTA per leaf with very uneven source counts,
  // so the launch's tail is its lightest leaves (tmpA is indexed by position
  // and scattered through this same list: results unchanged)
  std::stable_sort(p2m.begin(), p2m.end(), [&](int64_t a, int64_t c) {
    const int64_t ba = P->id_of[a], bc = P->id_of[c];
    return t.src_hi[ba] - t.src_lo[ba] > t.src_hi[bc] - t.src_lo[bc];
  });
  D.n_p2m = (int64_t)p2m.size();
  LB_TRY(upload(&D.p2m_leaves, p2m));
  if (src_range) LB_TRY(upload(&D.src_own, src_own));
  // X / W entries evaluated directly (lb_fmm_plan_set_xw; the lists below)
  const bool xw = P->xw_direct != 0;
  auto x_direct = [&](int64_t b) {
    const int64_t ntb = t.tgt_hi[b] - t.tgt_lo[b];
    return xw && t.is_leaf[b] && ntb > 0 && 5 * ntb <= 2 * (int64_t)nrep;
  };
  auto w_direct = [&](int64_t w) { return xw && t.is_leaf[w] && t.src_hi[w] - t.src_lo[w] <= (int64_t)nrep; };
  // Translations nobody reads are skipped (the reference computes them,
  // fmm.py:853-871, 913-935; the results at the targets are unchanged):
  //  * a box's multipole is NEEDED if it is a V-list source or a (non-direct)
  //    W-list member of any box with targets -- on every rank: the ranks'
  //    partial expansions are summed -- or if its parent's is; an M2M edge
  //    child -> parent exists only for needed parents (the root's and level
  //    1's expansions are never read);
  //  * a box's local expansion is NONZERO if it has V-list sources or
  //    (non-direct) X-list leaves, or its parent's is; an L2L edge parent ->
  //    child exists only for nonzero parents, and a level without any nonzero
  //    box gets its local expansions zeroed instead of computed.
  std::vector<uint8_t> need_up(nb, 0), nz_dn(nb, 0);
  for (int64_t b = 0; b < nb; ++b) {
    if (t.tgt_hi[b] <= t.tgt_lo[b]) continue;
    for (int64_t q = 0; q < t.vlist.size(b); ++q) need_up[t.vlist.row(b)[q]] = 1;
    if (t.is_leaf[b])
      for (int64_t q = 0; q < t.wlist.size(b); ++q) {
        const int64_t w = t.wlist.row(b)[q];
        if (!w_direct(w)) need_up[w] = 1;
      }
    bool dc = t.vlist.size(b) > 0;
    if (!dc && !x_direct(b))
      for (int64_t q = 0; q < t.xlist.size(b) && !dc; ++q) {
        const int64_t x = t.xlist.row(b)[q];
        dc = t.src_hi[x] > t.src_lo[x];
      }
    nz_dn[b] = dc ? 1 : 0;
  }
  std::vector<uint8_t> level_loc(t.nlev, 0);
  for (int l = 0; l < t.nlev; ++l)
    for (int64_t b : t.levels[l]) {
      const int64_t p = t.parent[b];
      if (l > 0 && nz_dn[p]) nz_dn[b] = 1;
      if (nz_dn[b] && own_id[b]) level_loc[l] = 1;
    }
  for (int l = 1; l < t.nlev; ++l)  // a needed parent needs its children
    for (int64_t b : t.levels[l])
      if (need_up[t.parent[b]]) need_up[b] = 1;
  D.level_loc.assign(level_loc.begin(), level_loc.end());
  std::vector<int64_t> uc, upar, dch, dpar, mpar, mch8;
  D.up_off.assign(1, 0);
  D.dn_off.assign(1, 0);
  D.up_par_off.assign(1, 0);
  {  // buckets per (level, octant), boxes in ascending id within a level
    std::vector<std::vector<int64_t>> bu(8), bd(8);
    for (int l = 0; l < t.nlev; ++l) {
      for (auto& v : bu) v.clear();
      for (auto& v : bd) v.clear();
      if (l > 0)
        for (int64_t b : t.levels[l]) {
          const int64_t s = S[b];
          const int oct = (int)octant[s];
          const int64_t p = t.parent[b];
          // fmm.py:855-859 (with a source range: subtrees holding owned sources)
          if (!t.is_leaf[p] && t.nsrc[p] > 0 && t.nsrc[b] > 0 && nsrc_own(b) > 0 && need_up[p]) bu[oct].push_back(b);
          // fmm.py:923-935 passes down to every child; children without targets
          // in their subtree never reach an L2T or a leaf, so they are skipped
          // (the results at the targets are unchanged; a plan whose targets are
          // one rank's rows skips most of the downward pass)
          if (own_id[b] && nz_dn[p]) bd[oct].push_back(b);
        }
      const int64_t ubase = (int64_t)uc.size();
      for (int oct = 0; oct < 8; ++oct) {
        for (int64_t b : bu[oct]) {
          uc.push_back(S[b]);
          upar.push_back(S[t.parent[b]]);
        }
        for (int64_t b : bd[oct]) {
          dch.push_back(S[b]);
          dpar.push_back(S[t.parent[b]]);
        }
        D.up_off.push_back((int64_t)uc.size());
        D.dn_off.push_back((int64_t)dch.size());
      }
      // surface M2M sum: this level's parents (slots ascending), each with the
      // positions of its children in the level's child list, octant order
      std::map<int64_t, int64_t> row;
      for (int64_t i = ubase; i < (int64_t)uc.size(); ++i) row.emplace(upar[i], 0);
      int64_t r = 0;
      for (auto& kv : row) {
        kv.second = r++;
        mpar.push_back(kv.first);
      }
      const size_t base = mch8.size();
      mch8.resize(base + 8 * row.size(), -1);
      for (int64_t i = ubase; i < (int64_t)uc.size(); ++i)
        mch8[base + 8 * row[upar[i]] + octant[uc[i]]] = i - ubase;
      D.up_par_off.push_back((int64_t)mpar.size());  // parents of level l's children
    }
  }
  LB_TRY(upload(&D.up_child, uc));
  LB_TRY(upload(&D.up_parent, upar));
  LB_TRY(upload(&D.dn_child, dch));
  LB_TRY(upload(&D.dn_parent, dpar));
  LB_TRY(upload(&D.up_par, mpar));
  LB_TRY(upload(&D.up_child8, mch8));
  LB_TRY(upload(&D.dn_off_dev, D.dn_off));
  LB_TRY(upload(&D.up_off_dev, D.up_off));
  mark("m2m/l2l");
  // M2L pairs grouped by canonical key, each group in target-slot order (the
  // walk below visits targets in slot order, so no sort is needed).  Lattice
  // offsets are looked up in a dense table; boxes are split into contiguous
  // chunks whose per-key counts place every pair deterministically.
  std::vector<int32_t> off_table(kOffW * kOffW * kOffW, -1);
  for (int d = 0; d < P->noff; ++d) {
    const int* v = &P->off_vec[3 * d];
    if (std::abs(v[0]) > kOffR || std::abs(v[1]) > kOffR || std::abs(v[2]) > kOffR)
      return fail(LB_ERR_ARG, "fmm: M2L lattice offset out of range");
    off_table[((v[0] + kOffR) * kOffW + (v[1] + kOffR)) * kOffW + (v[2] + kOffR)] = d;
  }
  if (P->tdev.v_idx) {
    LB_TRY(m2l_pairs_device(P, own_id, off_table));
  } else {
    std::vector<int64_t> vt_boxes;  // target boxes in slot order
    for (int64_t sl = 0; sl < nb; ++sl) {
      const int64_t b = P->id_of[sl];
      if (owned(b) > 0 && t.vlist.size(b) > 0) vt_boxes.push_back(b);
    }
    const int nk = P->ncanon;
    const int64_t nvt = (int64_t)vt_boxes.size();
    const int nchunk = (int)std::min<int64_t>(std::max<int64_t>(nvt, 1), 256);
    std::vector<int64_t> kcnt((size_t)nchunk * nk, 0);
    bool bad_off = false;
    auto pair_off = [&](int64_t b, int64_t src) {
      const int64_t dx = t.ijk[3 * src] - t.ijk[3 * b], dy = t.ijk[3 * src + 1] - t.ijk[3 * b + 1],
                    dz = t.ijk[3 * src + 2] - t.ijk[3 * b + 2];
      if (std::llabs(dx) > kOffR || std::llabs(dy) > kOffR || std::llabs(dz) > kOffR) return -1;
      return (int)off_table[((dx + kOffR) * kOffW + (dy + kOffR)) * kOffW + (dz + kOffR)];
    };
  #pragma omp parallel for schedule(static) reduction(|| : bad_off)
    for (int c = 0; c < nchunk; ++c) {
      for (int64_t i = nvt * c / nchunk; i < nvt * (c + 1) / nchunk; ++i) {
        const int64_t b = vt_boxes[i];
        for (int64_t q = 0; q < t.vlist.size(b); ++q) {
          const int d = pair_off(b, t.vlist.row(b)[q]);
          if (d < 0) { bad_off = true; continue; }
          ++kcnt[(size_t)c * nk + P->off_key[d]];
        }
      }
    }
    if (bad_off) return fail(LB_ERR_ARG, "fmm: V-list offset without an M2L operator");
    D.v_key_pair_off.assign(nk + 1, 0);
    for (int k = 0; k < nk; ++k) {
      int64_t tot = 0;
      for (int c = 0; c < nchunk; ++c) tot += kcnt[(size_t)c * nk + k];
      D.v_key_pair_off[k + 1] = D.v_key_pair_off[k] + tot;
    }
    const int64_t npairs = D.v_key_pair_off[nk];
    std::vector<int64_t> kpos((size_t)nchunk * nk);  // chunk c's first slot in key k
    for (int k = 0; k < nk; ++k) {
      int64_t at = D.v_key_pair_off[k];
      for (int c = 0; c < nchunk; ++c) {
        kpos[(size_t)c * nk + k] = at;
        at += kcnt[(size_t)c * nk + k];
      }
    }
    std::vector<int64_t> vsrc(npairs), vtgt(npairs);
    std::vector<int32_t> voff(npairs);
    std::vector<double> vscale(npairs);
  #pragma omp parallel for schedule(static)
    for (int c = 0; c < nchunk; ++c) {
      int64_t* pos = &kpos[(size_t)c * nk];
      for (int64_t i = nvt * c / nchunk; i < nvt * (c + 1) / nchunk; ++i) {
        const int64_t b = vt_boxes[i];
        const double inv_h = 1.0 / (t.half / std::ldexp(1.0, t.level[b]));  // fmm.py:879
        for (int64_t q = 0; q < t.vlist.size(b); ++q) {
          const int64_t src = t.vlist.row(b)[q];
          const int d = pair_off(b, src);
          const int64_t at = pos[P->off_key[d]]++;
          vsrc[at] = S[src];
          vtgt[at] = S[b];
          voff[at] = d;
          vscale[at] = inv_h;
        }
      }
    }
    mark("m2l pairs");
    std::vector<int64_t> vtgts, tpoff{0};
    D.v_key_tgt_off.assign(1, 0);
    D.max_key_pairs = 0;
    for (int k = 0; k < nk; ++k) {
      const int64_t a = D.v_key_pair_off[k], e = D.v_key_pair_off[k + 1];
      for (int64_t i = a; i < e; ++i) {
        if (i == a || vtgt[i] != vtgt[i - 1]) {
          if (i > a) tpoff.push_back(i);
          vtgts.push_back(vtgt[i]);
        }
      }
      if (e > a) tpoff.push_back(e);
      D.v_key_tgt_off.push_back((int64_t)vtgts.size());
      D.max_key_pairs = std::max<int64_t>(D.max_key_pairs, e - a);
    }
    mark("m2l tgts");
    LB_TRY(upload(&D.v_src, vsrc));
    LB_TRY(upload(&D.v_tgts, vtgts));
    LB_TRY(upload(&D.v_tgt_pair_off, tpoff));
    D.v_tpoff_host = tpoff;
    LB_TRY(upload(&D.v_off_idx, voff));
    LB_TRY(upload(&D.v_scale, vscale));
  }
  mark("m2l upload");
  // X list (fmm.py:891-911): boxes with sourceful X entries; leaf stage
  // (fmm.py:940-988): target leaves, their U (with sources) and W lists.
  // Count / scan / fill, parallel over boxes, same order as a serial walk.
  // With xw_direct (lb_fmm_plan_set_xw) two of the reference's approximate
  // interactions are evaluated exactly where that is also cheaper:
  //  * an X-list entry (target box b, source leaf x) of a LEAF b with few
  //    targets (2.5 nt(b) <= nrep): x's sources act directly on b's targets
  //    (joins b's U list) instead of on b's nrep check points;
  //  * a W-list entry (target leaf b, box w) whose w is a leaf with at most
  //    nrep sources: w's sources act directly (joins b's U list) instead of
  //    w's nrep equivalent charges.
  // Appended after the reference's U entries, X first, in list order.
  std::vector<int64_t> xcnt(nb, 0), ucnt(nb, 0), wcnt(nb, 0);
  std::vector<uint8_t> is_tl(nb, 0);
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t b = 0; b < nb; ++b) {
    if (!own_id[b]) continue;  // as for M2L
    const bool xd = x_direct(b);
    int64_t nx = 0;
    for (int64_t q = 0; q < t.xlist.size(b); ++q) {
      const int64_t x = t.xlist.row(b)[q];
      nx += t.src_hi[x] > t.src_lo[x] ? 1 : 0;
    }
    if (!xd) xcnt[b] = nx;
    if (!t.is_leaf[b]) continue;
    is_tl[b] = 1;
    if (xd) ucnt[b] += nx;
    for (int64_t q = 0; q < t.ulist.size(b); ++q) {
      const int64_t u = t.ulist.row(b)[q];
      ucnt[b] += t.src_hi[u] > t.src_lo[u] ? 1 : 0;
    }
    for (int64_t q = 0; q < t.wlist.size(b); ++q) {
      const int64_t w = t.wlist.row(b)[q];
      if (w_direct(w)) ucnt[b] += t.src_hi[w] > t.src_lo[w] ? 1 : 0;
      else ++wcnt[b];
    }
  }
  std::vector<int64_t> xb, xo{0}, tl, uo{0}, wo{0}, xpos(nb), upos(nb), wpos(nb);
  for (int64_t b = 0; b < nb; ++b) {
    xpos[b] = xo.back();
    if (xcnt[b] > 0) {
      xb.push_back(S[b]);
      xo.push_back(xo.back() + xcnt[b]);
    }
    upos[b] = uo.back();
    wpos[b] = wo.back();
    if (is_tl[b]) {
      tl.push_back(S[b]);
      uo.push_back(uo.back() + ucnt[b]);
      wo.push_back(wo.back() + wcnt[b]);
    }
  }
  std::vector<int64_t> xl(xo.back()), ul(uo.back()), wl(wo.back());
#pragma omp parallel for schedule(dynamic, 1024)
  for (int64_t b = 0; b < nb; ++b) {
    if (xcnt[b] > 0) {
      int64_t o = xpos[b];
      for (int64_t q = 0; q < t.xlist.size(b); ++q) {
        const int64_t x = t.xlist.row(b)[q];
        if (t.src_hi[x] > t.src_lo[x]) xl[o++] = S[x];
      }
    }
    if (is_tl[b]) {
      int64_t o = upos[b];
      for (int64_t q = 0; q < t.ulist.size(b); ++q) {
        const int64_t u = t.ulist.row(b)[q];
        if (t.src_hi[u] > t.src_lo[u]) ul[o++] = S[u];
      }
      if (x_direct(b)) {
        for (int64_t q = 0; q < t.xlist.size(b); ++q) {
          const int64_t x = t.xlist.row(b)[q];
          if (t.src_hi[x] > t.src_lo[x]) ul[o++] = S[x];
        }
      }
      int64_t ow = wpos[b];
      for (int64_t q = 0; q < t.wlist.size(b); ++q) {
        const int64_t w = t.wlist.row(b)[q];
        if (w_direct(w)) {
          if (t.src_hi[w] > t.src_lo[w]) ul[o++] = S[w];
        } else {
          wl[ow++] = S[w];
        }
      }
    }
  }
  D.n_x = (int64_t)xb.size();
  LB_TRY(upload(&D.x_boxes, xb));
  LB_TRY(upload(&D.x_off, xo));
  LB_TRY(upload(&D.x_leaves, xl));
  mark("x list");
  D.n_tleaf = (int64_t)tl.size();
  mark("leaf lists");
  // work items: a leaf's virtual source list [U sources | own DE set | W sets]
  // is cut into segments of at most ~2^20 (target, source) pairs, so no block
  // is the kernel's critical path (measured: SMs idle half of the leaf stage
  // on config 3 without this); split leaves reduce their partials in order
  {
    std::vector<int64_t> items, islot, sleaf, srange, weight;
    int64_t slots = 0;
    for (int64_t li = 0; li < D.n_tleaf; ++li) {
      const int64_t b = P->id_of[tl[li]];
      const int64_t ntl = t.tgt_hi[b] - t.tgt_lo[b];
      int64_t vtot = (P->rep == 0 ? nrep : 0) + (wo[li + 1] - wo[li]) * (int64_t)nrep;
      for (int64_t q = uo[li]; q < uo[li + 1]; ++q) {
        const int64_t u = P->id_of[ul[q]];
        vtot += t.src_hi[u] - t.src_lo[u];
      }
      const int64_t seg = std::max<int64_t>(1024, ((int64_t)1 << 20) / std::max<int64_t>(ntl, 1));
      const int64_t nseg = std::max<int64_t>(1, ceil_div(vtot, seg));
      if (nseg > 1) {
        sleaf.push_back(li);
        srange.push_back((int64_t)(items.size() / 4));
        srange.push_back((int64_t)(items.size() / 4) + nseg);
      }
      for (int64_t k = 0; k < nseg; ++k) {
        items.push_back(li);
        items.push_back(k * seg);
        items.push_back(k + 1 == nseg ? vtot : (k + 1) * seg);
        items.push_back(-1);
        weight.push_back(std::max<int64_t>(ntl, 1) * ((k + 1 == nseg ? vtot : (k + 1) * seg) - k * seg));
        islot.push_back(nseg == 1 ? -1 : slots);
        if (nseg > 1) slots += ntl;
      }
    }
    D.n_items = (int64_t)(items.size() / 4);
    D.n_split = (int64_t)sleaf.size();
    D.part_doubles = slots;
    D.part_width = -1;
    LB_TRY(upload(&D.leaf_items, items));
    LB_TRY(upload(&D.leaf_item_slot, islot));
    // launch order: heaviest item first (block i runs item order[i]), so the
    // stage does not end on a few 2^20-pair items that started last; every
    // item still writes its own outputs / slots, results unchanged
    std::vector<int64_t> order(D.n_items);
    for (int64_t i = 0; i < D.n_items; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t c) { return weight[a] > weight[c]; });
    LB_TRY(upload(&D.leaf_order, order));
    LB_TRY(upload(&D.split_leaf, sleaf));
    LB_TRY(upload(&D.split_item_off, srange));  // [first item, end) per split leaf
  }
  mark("leaf items");
  LB_TRY(upload(&D.t_leaves, tl));
  LB_TRY(upload(&D.u_off, uo));
  LB_TRY(upload(&D.u_list, ul));
  LB_TRY(upload(&D.w_off, wo));
  LB_TRY(upload(&D.w_list, wl));
  // octant per slot is needed by the grid tensor kernel: keep it in bsrc's
  // companion buffer
  D.btgt_oct = doct;
  D.level_slot_off = level_slot_off;
  mark("leaf upload");
  LB_CUDA(cudaStreamSynchronize(0));  // the setup kernels above ran on the legacy stream
  D.ready = true;
  return LB_OK;
}

int ensure_work(lb_fmm_plan* P, int nd) {
  // work arrays are sized for the largest density chunk seen so far and never
  // shrunk: callers alternate nd (the operator apply uses 1 then 3), and a
  // cudaFree/cudaMalloc pair per call would serialise the device
  FmmDevice& D = P->dev;
  if (D.nd_alloc >= nd) return LB_OK;
  nd = std::max(nd, std::min(4, 2 * std::max(D.nd_alloc, 1)));
  if (D.loc != D.dc) cudaFree(D.loc);  // grid: loc aliases dc
  cudaFree(D.cs); cudaFree(D.vs); cudaFree(D.up); cudaFree(D.dc);
  cudaFree(D.cs_own); cudaFree(D.vs_own);
  D.cs_own = D.vs_own = nullptr;
  cudaFree(D.tmpA); cudaFree(D.tmpB); cudaFree(D.tout);
  D.cs = D.vs = D.up = D.dc = D.loc = D.tmpA = D.tmpB = D.tout = nullptr;
  const FmmTree& t = P->tree;
  const int64_t nb = t.nbox(), nrep = P->nrep;
  // GEMM staging: the largest of (P2M leaves, any level/octant group, M2L chunk)
  int64_t cols = std::max<int64_t>(D.n_p2m, 1);
  for (size_t i = 0; i + 8 < D.up_off.size(); i += 8) cols = std::max(cols, D.up_off[i + 8] - D.up_off[i]);
  for (size_t i = 0; i + 1 < D.dn_off.size(); ++i) cols = std::max(cols, D.dn_off[i + 1] - D.dn_off[i]);
  const int64_t m2l_cap = std::max<int64_t>(1, std::min<int64_t>(D.max_key_pairs, (int64_t)1 << 17));
  cols = std::max(cols, m2l_cap);
  D.tmp_cols = cols;
  cudaError_t e = cudaSuccess;
  auto A = [&](double** p, int64_t n) { if (e == cudaSuccess) e = cudaMalloc((void**)p, std::max<int64_t>(n, 2) * 8); };
  A(&D.cs, (int64_t)nd * t.ns);
  A(&D.vs, (int64_t)nd * t.ns * 3);
  if (D.src_own) {
    A(&D.cs_own, (int64_t)nd * t.ns);
    A(&D.vs_own, (int64_t)nd * t.ns * 3);
  }
  A(&D.up, nb * nd * nrep);
  A(&D.dc, nb * nd * nrep);
  if (P->rep == 0) A(&D.loc, nb * nd * nrep);
  A(&D.tmpA, cols * nd * nrep);
  A(&D.tmpB, cols * nd * nrep);
  A(&D.tout, (int64_t)nd * t.nt * 10);
  if (e != cudaSuccess) return fail(LB_ERR_CUDA, std::string("fmm work arrays: ") + cudaGetErrorString(e));
  if (P->rep == 1) D.loc = D.dc;  // grid: local = dcheck (fmm.py:918)
  D.nd_alloc = nd;
  return LB_OK;
}

// tcgen05 M2L state: A packs of every canonical matrix for the current slice
// count, column-pack capacity for the largest M2L chunk of nd densities
int ensure_oz(lb_fmm_plan* P, int nd, cudaStream_t st) {
  FmmDevice& D = P->dev;
  const int S = P->m2l_slices, nrep = P->nrep;
  if (S <= 0) return LB_OK;
  if (nrep > 2048) return fail(LB_ERR_ARG, "tensor-core M2L needs nrep <= 2048 (set m2l slices to 0)");
  if (D.oz_S != S) {
    cudaFree(D.oz_a);
    cudaFree(D.oz_rs);
    D.oz_a = nullptr;
    D.oz_rs = nullptr;
    D.oz_S = 0;
    const int mpad = ceil_div(nrep, oz::kBM) * oz::kBM;
    LB_CUDA(cudaMalloc((void**)&D.oz_a, oz::pack_rows_bytes(nrep, S) * std::max(P->ncanon, 1)));
    LB_CUDA(cudaMalloc((void**)&D.oz_rs, sizeof(double) * mpad * std::max(P->ncanon, 1)));
    if (P->ncanon > 0) {
      oz::pack_rows_kernel<<<dim3((unsigned)mpad, (unsigned)P->ncanon), 256, 0, st>>>(D.canon, nrep, S, D.oz_a,
                                                                                       D.oz_rs);
      LB_CHECK_LAUNCH();
    }
    D.oz_S = S;
  }
  const int64_t need = D.tmp_cols * nd;
  if (D.oz_cols < need) {
    cudaFree(D.oz_b);
    cudaFree(D.oz_cs);
    D.oz_b = nullptr;
    D.oz_cs = nullptr;
    D.oz_cols = 0;
    LB_CUDA(cudaMalloc((void**)&D.oz_b, oz::pack_cols_bytes_max(nrep, need)));
    LB_CUDA(cudaMalloc((void**)&D.oz_cs, sizeof(double) * need));
    D.oz_cols = need;
  }
  return LB_OK;
}


// Y[:, cols] = alpha * A * X[:, cols] for contiguous column blocks (the
// M2L's second low-rank factor, L2L's pinv_dn): dgemm_cols.cuh
int gemm_contig(const double* A, int lda, int M, int K, const double* X, int64_t ldx, double* Y,
                int64_t ldy, int64_t ncols, double alpha, cudaStream_t st) {
  dg::Args a{};
  a.A = A; a.lda = lda; a.M = M; a.K = K; a.S = 1; a.nd = 1;
  a.X = X; a.ldx = ldx; a.Y = Y; a.ldy = ldy; a.alpha = alpha; a.add = 0; a.nq = ncols;
  LB_DG(dg::gemm_cols(a, ncols, 1, st));
  return LB_OK;
}

// low-rank M2L: device copies of the factors and the rank-sized staging
int ensure_lowrank(lb_fmm_plan* P, int nd) {
  FmmDevice& D = P->dev;
  if (!D.lr_a) {
    LB_CUDA(cudaMalloc((void**)&D.lr_a, sizeof(double) * std::max<size_t>(P->lr_a_host.size(), 1)));
    LB_CUDA(cudaMalloc((void**)&D.lr_b, sizeof(double) * std::max<size_t>(P->lr_b_host.size(), 1)));
    LB_CUDA(cudaMemcpy(D.lr_a, P->lr_a_host.data(), sizeof(double) * P->lr_a_host.size(), cudaMemcpyHostToDevice));
    LB_CUDA(cudaMemcpy(D.lr_b, P->lr_b_host.data(), sizeof(double) * P->lr_b_host.size(), cudaMemcpyHostToDevice));
    D.lo_ready = false;
  }
  const int nk = P->ncanon, nrep = P->nrep;
  if (!D.lr_ap) {  // A_k in DMMA fragment order for the fused second factor (m2l_fused.cuh)
    D.lr_ap_off.assign(nk + 1, 0);
    for (int k = 0; k < nk; ++k)
      D.lr_ap_off[k + 1] = D.lr_ap_off[k] + (int64_t)m2lf::packed_doubles(nrep, P->lr_rank[k]);
    std::vector<double> ap(std::max<int64_t>(D.lr_ap_off[nk], 1));
#pragma omp parallel for schedule(dynamic, 1)
    for (int k = 0; k < nk; ++k)
      m2lf::pack_a(P->lr_a_host.data() + P->lr_off[k] * nrep, nrep, P->lr_rank[k], ap.data() + D.lr_ap_off[k]);
    LB_TRY(upload(&D.lr_ap, ap));
  }
  if (!D.lo_ready) {
    // pair arrays back on the host once (the device plan build leaves them on the device)
    const int64_t np = D.v_key_pair_off[nk];
    std::vector<int64_t> vsrc(np);
    std::vector<int32_t> voff(np);
    std::vector<double> vsc(np);
    if (np) {
      LB_CUDA(cudaMemcpy(vsrc.data(), D.v_src, 8 * np, cudaMemcpyDeviceToHost));
      LB_CUDA(cudaMemcpy(voff.data(), D.v_off_idx, 4 * np, cudaMemcpyDeviceToHost));
      LB_CUDA(cudaMemcpy(vsc.data(), D.v_scale, 8 * np, cudaMemcpyDeviceToHost));
    }
    // B_k P_d for every offset d: T = B_k x[perm_inv] = (B_k[:, perm]) x
    std::vector<int64_t> bp_off(P->noff + 1, 0);
    for (int d = 0; d < P->noff; ++d) bp_off[d + 1] = bp_off[d] + (int64_t)P->lr_rank[P->off_key[d]] * nrep;
    std::vector<double> bp(std::max<int64_t>(bp_off.back(), 1));
#pragma omp parallel for schedule(dynamic, 4)
    for (int d = 0; d < P->noff; ++d) {
      const int k = P->off_key[d], r = P->lr_rank[k];
      const double* B = P->lr_b_host.data() + P->lr_off[k] * nrep;
      const int32_t* pm = P->off_perm.data() + (int64_t)d * nrep;
      double* o = bp.data() + bp_off[d];
      for (int a = 0; a < r; ++a)
        for (int j = 0; j < nrep; ++j) o[(int64_t)a * nrep + j] = B[(int64_t)a * nrep + pm[j]];
    }
    // every key's pairs by offset (stable): the first factor's batches
    std::vector<int64_t> lsrc(np), ltcol(np), boff, aoff;
    std::vector<double> lsc(np);
    D.lo_key_batch.assign(nk + 1, 0);
    D.lo_key_maxgrp.assign(nk, 0);
    std::vector<int64_t> cnt(P->noff);
    for (int k = 0; k < nk; ++k) {
      const int64_t p0 = D.v_key_pair_off[k], p1 = D.v_key_pair_off[k + 1];
      D.lo_key_batch[k] = (int64_t)boff.size();
      std::fill(cnt.begin(), cnt.end(), 0);
      for (int64_t i = p0; i < p1; ++i) ++cnt[voff[i]];
      std::vector<int64_t> at(P->noff);
      int64_t pos = p0;
      for (int d = 0; d < P->noff; ++d) {
        at[d] = pos;
        if (cnt[d]) {
          boff.push_back(pos);
          aoff.push_back(bp_off[d]);
          D.lo_key_maxgrp[k] = std::max(D.lo_key_maxgrp[k], cnt[d]);
        }
        pos += cnt[d];
      }
      boff.push_back(p1);
      aoff.push_back(0);  // keeps aoff aligned with boff (nbatch + 1 entries per key)
      for (int64_t i = p0; i < p1; ++i) {
        const int64_t j = at[voff[i]]++;
        lsrc[j] = vsrc[i];
        ltcol[j] = i - p0;
        lsc[j] = vsc[i];
      }
    }
    D.lo_key_batch[nk] = (int64_t)boff.size();
    {  // the single-launch form: every key's batches, T of key k at tbase1[k] * nd
      std::vector<int64_t> gb, ga, gy;
      std::vector<int32_t> gm;
      D.lo_tbase1.assign(nk + 1, 0);
      D.lo_gmaxgrp = 0;
      D.lo_rmax = 0;
      for (int k = 0; k < nk; ++k) {
        const int64_t p0 = D.v_key_pair_off[k], p1 = D.v_key_pair_off[k + 1];
        const int r = P->lr_rank[k];
        D.lo_tbase1[k + 1] = D.lo_tbase1[k] + (p1 - p0) * m2lf::tstride(r);
        if (p1 == p0) continue;
        for (int64_t e = D.lo_key_batch[k]; e + 1 < D.lo_key_batch[k + 1]; ++e) {
          gb.push_back(boff[e]);
          ga.push_back(aoff[e]);
          gy.push_back(D.lo_tbase1[k]);
          gm.push_back(r);
        }
        D.lo_gmaxgrp = std::max(D.lo_gmaxgrp, D.lo_key_maxgrp[k]);
        D.lo_rmax = std::max(D.lo_rmax, r);
      }
      D.lo_gbatch = (int64_t)gm.size();
      gb.push_back(np);
      D.lo_gm_host = gm;
      D.lo_gb_host = gb;
      D.lo_gb0 = gb.front();  // q of the launch counts from the first nonempty key's pairs
      cudaFree(D.lo_gboff); cudaFree(D.lo_gaoff); cudaFree(D.lo_gyoff); cudaFree(D.lo_gm);
      D.lo_gboff = D.lo_gaoff = D.lo_gyoff = nullptr;
      D.lo_gm = nullptr;
      LB_TRY(upload(&D.lo_gboff, gb));
      LB_TRY(upload(&D.lo_gaoff, ga));
      LB_TRY(upload(&D.lo_gyoff, gy));
      LB_TRY(upload(&D.lo_gm, gm));
    }

    cudaFree(D.lr_bp); cudaFree(D.lo_src); cudaFree(D.lo_tcol); cudaFree(D.lo_scale);
    cudaFree(D.lo_boff); cudaFree(D.lo_aoff);
    D.lr_bp = D.lo_scale = nullptr;
    D.lo_src = D.lo_tcol = D.lo_boff = D.lo_aoff = nullptr;
    LB_TRY(upload(&D.lr_bp, bp));
    LB_TRY(upload(&D.lo_src, lsrc));
    LB_TRY(upload(&D.lo_tcol, ltcol));
    LB_TRY(upload(&D.lo_scale, lsc));
    LB_TRY(upload(&D.lo_boff, boff));
    LB_TRY(upload(&D.lo_aoff, aoff));
    for (int i = 0; i < 5; ++i) {
      cudaFree(D.lo_units[i]);
      cudaFree(D.lo_tiles[i]);
      cudaFree(D.lo_unit_key[i]);
      D.lo_units[i] = nullptr;
      D.lo_tiles[i] = nullptr;
      D.lo_unit_key[i] = nullptr;
    }
    cudaFree(D.lo_keytab); cudaFree(D.lo_rt_tgt); cudaFree(D.lo_rt_off); cudaFree(D.lo_rt_grp);
    D.lo_keytab = D.lo_rt_tgt = D.lo_rt_off = D.lo_rt_grp = nullptr;
    D.lo_ready = true;
  }
  if (nd < 1 || nd > 4) return fail(LB_ERR_ARG, "fmm: density chunk outside [1, 4]");
  if (!D.lo_fit_done) {  // the cube-symmetry permutations in closed form (m2l_fused.cuh)
    std::vector<int32_t> aff;
    std::vector<uint32_t> coords;
    std::vector<uint16_t> lut;
    int m = 0;
    if (m2lf::fit_symmetries(P->pts.data(), nrep, P->off_perm.data(), P->noff, aff, coords, lut, m)) {
      LB_TRY(upload(&D.lo_aff, aff));
      LB_TRY(upload(&D.lo_coords, coords));
      LB_TRY(upload(&D.lo_lut, lut));
      D.lo_lut_n = m * m * m;
    }
    if (std::getenv("LB_FMM_DEBUG"))
      std::fprintf(stderr, "fmm: closed-form M2L permutations %s (nrep %d, %d offsets, lattice %d^3)\n",
                   D.lo_aff ? "fitted" : "NOT fitted, table lookups", nrep, P->noff, m);
    D.lo_fit_done = true;
  }
  if (!D.lo_carry) {  // carry pool of the multi-pass groups (m2l_fused.cuh)
    int dev = 0, sms = 0;
    LB_CUDA(cudaGetDevice(&dev));
    LB_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    D.lo_carry_slots = m2lf::carry_slots(sms);
    LB_CUDA(cudaMalloc((void**)&D.lo_carry,
                       sizeof(double) * (size_t)D.lo_carry_slots * m2lf::kMaxNd * P->nrep));
    LB_CUDA(cudaMalloc((void**)&D.lo_carry_flag, sizeof(unsigned) * (size_t)D.lo_carry_slots));
    LB_CUDA(cudaMemset(D.lo_carry_flag, 0, sizeof(unsigned) * (size_t)D.lo_carry_slots));
  }
  if (!D.lo_keytab) {  // per key: A_k offsets, T offset per density, first pair, rank (m2l_fused.cuh)
    std::vector<int64_t> ktab(5 * (size_t)std::max(nk, 1), 0);
    for (int k = 0; k < nk; ++k) {
      ktab[5 * k] = D.lr_ap_off[k];
      ktab[5 * k + 1] = P->lr_off[k] * nrep;
      ktab[5 * k + 2] = D.lo_tbase1[k];
      ktab[5 * k + 3] = D.v_key_pair_off[k];
      ktab[5 * k + 4] = P->lr_rank[k];
    }
    LB_TRY(upload(&D.lo_keytab, ktab));
    // every target's (target, key) groups by ascending key, for the ordered
    // reduction of the groups' partial sums into the check values
    const int64_t ng = D.v_key_tgt_off[nk];
    std::vector<int64_t> vt(std::max<int64_t>(ng, 1));
    if (ng) LB_CUDA(cudaMemcpy(vt.data(), D.v_tgts, 8 * ng, cudaMemcpyDeviceToHost));
    std::vector<int64_t> order(ng);
    for (int64_t i = 0; i < ng; ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](int64_t a, int64_t b) { return vt[a] < vt[b]; });
    std::vector<int64_t> rt_tgt, rt_off{0};
    for (int64_t i = 0; i < ng; ++i) {  // group indices ascend with the key: the stable sort keeps key order
      if (i == 0 || vt[order[i]] != vt[order[i - 1]]) {
        if (i) rt_off.push_back(i);
        rt_tgt.push_back(vt[order[i]]);
      }
    }
    rt_off.push_back(ng);
    if (ng == 0) rt_off.assign(1, 0);
    D.lo_rt_n = (int64_t)rt_tgt.size();
    LB_TRY(upload(&D.lo_rt_tgt, rt_tgt));
    LB_TRY(upload(&D.lo_rt_off, rt_off));
    LB_TRY(upload(&D.lo_rt_grp, order));
  }
  if (!D.lo_units[nd]) {  // units of whole target groups, <= one pass of columns where possible
    // Units in (key, group) order are cut into batches whose groups' partial
    // sums fit the scratch buffer (LB_M2L_PART_MB, default 3072 MB); a
    // batch's units run in ONE launch, the highest ranks first, and are then
    // reduced into the check values before the next batch starts.
    static const int64_t cap_bytes = [] {
      const char* e = std::getenv("LB_M2L_PART_MB");
      const int64_t mb = e ? std::atoll(e) : 3072;
      return std::max<int64_t>(mb, 16) << 20;
    }();
    const int64_t cap_groups = std::max<int64_t>(1, cap_bytes / ((int64_t)nd * nrep * 8));
    struct U { int64_t a, b; int32_t key; };
    std::vector<U> us;
    for (int k = 0; k < nk; ++k) {
      const int64_t g0 = D.v_key_tgt_off[k], g1 = D.v_key_tgt_off[k + 1];
      int64_t ub = g0, cols = 0;
      for (int64_t gi = g0; gi < g1; ++gi) {
        const int64_t c = (D.v_tpoff_host[gi + 1] - D.v_tpoff_host[gi]) * nd;
        if (gi > ub && cols + c > m2lf::pass_cols(nd)) {
          us.push_back({ub, gi, (int32_t)k});
          ub = gi;
          cols = 0;
        }
        cols += c;
      }
      if (g1 > ub) us.push_back({ub, g1, (int32_t)k});
    }
    std::vector<int64_t>& bo = D.lo_batch_off[nd];   // per batch: first unit; + end
    std::vector<int64_t>& bg = D.lo_batch_grp[nd];   // per batch: first group; + end
    bo.assign(1, 0);
    bg.assign(1, us.empty() ? 0 : us.front().a);
    int64_t maxg = 1;
    for (size_t i = 0; i < us.size(); ++i) {
      if (us[i].b - bg.back() > cap_groups && (int64_t)i > bo.back()) {
        bo.push_back((int64_t)i);
        bg.push_back(us[i].a);
      }
      maxg = std::max(maxg, us[i].b - bg.back());
    }
    bo.push_back((int64_t)us.size());
    bg.push_back(us.empty() ? 0 : us.back().b);
    for (size_t bi = 0; bi + 1 < bo.size(); ++bi)
      std::stable_sort(us.begin() + bo[bi], us.begin() + bo[bi + 1], [&](const U& x, const U& y) {
        return P->lr_rank[x.key] > P->lr_rank[y.key];
      });
    // one 64-byte record per unit (m2l_fused.cuh)
    std::vector<int64_t> urec;
    urec.reserve(m2lf::kRec * us.size());
    for (const U& u : us) {
      const int k = u.key, r = P->lr_rank[k];
      const int64_t pa = D.v_tpoff_host[u.a], pe = D.v_tpoff_host[u.b];
      urec.push_back(D.lr_ap_off[k]);
      urec.push_back(P->lr_off[k] * nrep);
      urec.push_back(D.lo_tbase1[k] * nd + (pa - D.v_key_pair_off[k]) * nd * m2lf::tstride(r));
      urec.push_back(r);
      urec.push_back(u.a);
      urec.push_back(u.b - u.a);
      urec.push_back(pa);
      urec.push_back(pe);
    }
    LB_TRY(upload(&D.lo_units[nd], urec));
    const int64_t need_part = maxg * nd * nrep;
    if (D.lo_part_cap < need_part) {
      cudaFree(D.lo_part);
      D.lo_part = nullptr;
      LB_CUDA(cudaMalloc((void**)&D.lo_part, sizeof(double) * need_part));
      D.lo_part_cap = need_part;
    }
    // the first factor's flat tile list (m2l_first.cuh): (batch, column tile),
    // the highest ranks first so the last wave holds the light tiles
    std::vector<std::pair<int32_t, int32_t>> tl;
    for (int64_t z = 0; z < D.lo_gbatch; ++z) {
      const int64_t cols = (D.lo_gb_host[z + 1] - D.lo_gb_host[z]) * nd;
      for (int64_t c = 0; c * m2l1::kBN < cols; ++c) tl.emplace_back((int32_t)z, (int32_t)c);
    }
    std::stable_sort(tl.begin(), tl.end(), [&](const auto& a, const auto& b) {
      return D.lo_gm_host[a.first] > D.lo_gm_host[b.first];
    });
    std::vector<int32_t> flat;
    flat.reserve(2 * tl.size());
    for (const auto& e : tl) {
      flat.push_back(e.first);
      flat.push_back(e.second);
    }
    D.lo_ntiles[nd] = (int64_t)tl.size();
    LB_TRY(upload(&D.lo_tiles[nd], flat));
  }
  int64_t need = std::max<int64_t>(1, D.lo_tbase1[nk] * nd);  // T of every key at once
  if (D.lr_t_cap < need) {

    cudaFree(D.lr_t);
    D.lr_t = nullptr;
    LB_CUDA(cudaMalloc((void**)&D.lr_t, sizeof(double) * need));
    // the fused path's T columns are padded to whole k-steps; the pad rows are
    // never written and must read as zero (m2l_fused.cuh)
    LB_CUDA(cudaMemset(D.lr_t, 0, sizeof(double) * need));
    D.lr_t_cap = need;
  }
  return LB_OK;
}

template <int ND>
int apply_chunk(lb_fmm_plan* P, int d0, uint32_t cmask, uint32_t dmask, const double* charges,
                const double* dipoles, int level, double* pot, double* grad, double* hess,
                cudaStream_t st, std::vector<cudaEvent_t>& ev, const double* proj_nrm = nullptr,
                double* proj_out = nullptr, const double* proj_snrm = nullptr) {
  FmmTree& t = P->tree;
  FmmDevice& D = P->dev;
  const int nrep = P->nrep;
  const int64_t nb = t.nbox();
  const bool surface = P->rep == 0;
  const int n = P->m;
  const unsigned dm_chunk = (dmask >> d0) & ((1u << ND) - 1u);  // the chunk's densities with dipoles
  const bool hd = dm_chunk != 0;
  auto mark = [&](int i) { if (!ev.empty()) cudaEventRecord(ev[i], st); };
  mark(0);
  // gather into sorted source order
  if (t.ns > 0) {
    gather_sources_kernel<<<(unsigned)ceil_div(t.ns, 256), 256, 0, st>>>(
        charges, dipoles, D.src_sorted, t.ns, ND, d0, cmask, dmask, D.cs, D.vs);
    LB_CHECK_LAUNCH();
  }
  LB_CUDA(cudaMemsetAsync(D.up, 0, sizeof(double) * nb * ND * nrep, st));
  LB_CUDA(cudaMemsetAsync(D.dc, 0, sizeof(double) * nb * ND * nrep, st));
  // P2M reads the owned sources only when a source range is set
  const double* p2m_cs = D.cs;
  const double* p2m_vs = D.vs;
  if (D.src_own && t.ns > 0) {
    mask_sources_kernel<<<(unsigned)ceil_div(t.ns, 256), 256, 0, st>>>(D.cs, D.vs, D.src_own, t.ns, ND,
                                                                       D.cs_own, D.vs_own);
    LB_CHECK_LAUNCH();
    p2m_cs = D.cs_own;
    p2m_vs = D.vs_own;
  }
  // ---- P2M (fmm.py:823-852)
  if (D.n_p2m > 0) {
    if (surface) {
      LB_TRY(launch_lattice<ND>((unsigned)D.n_p2m, st, D.p2m_leaves, nullptr, nullptr, 1, D.bctr, D.bhalf,
                                D.bsrc, D.spos, p2m_cs, p2m_vs, t.ns, (int)dm_chunk, D.pts, nrep, P->uc_scale, 1,
                                D.tmpA, 0, 0));
      // upward[b] = pinv_up @ (h phi) straight into the leaves' slots (fmm.py:852)
      dg::Args a{};
      a.A = D.pinv_up; a.lda = nrep; a.M = nrep; a.K = nrep; a.S = 1; a.nd = ND;
      a.X = D.tmpA; a.ldx = nrep; a.Y = D.up; a.ldy = nrep; a.out = D.p2m_leaves;
      a.alpha = 1.0; a.add = 0; a.nq = D.n_p2m;
      LB_DG(dg::gemm_cols(a, D.n_p2m * ND, 1, st));
    } else {
      p2m_grid_kernel<ND><<<(unsigned)D.n_p2m, 256, 0, st>>>(D.p2m_leaves, D.bctr, D.bhalf, D.bsrc,
                                                             D.spos, p2m_cs, p2m_vs, t.ns, hd ? 1 : 0, n,
                                                             D.vinv, D.up);
      LB_CHECK_LAUNCH();
    }
  }
  mark(1);
  // ---- M2M (fmm.py:853-871), deepest level first, octants in order
  const size_t grid_smem = sizeof(double) * 2 * nrep;
  for (int l = t.nlev - 1; l >= 1; --l) {
    if (surface) {
      // children of level l: m2m[octant] @ up[child] in 8 octant batches into
      // the staging, then every parent sums its children in octant order
      // (fmm.py:853-871; deterministic, no atomics)
      const int64_t u0 = D.up_off[8 * l], u1 = D.up_off[8 * l + 8];
      if (u1 > u0) {
        int64_t mx = 0;
        for (int oct = 0; oct < 8; ++oct) mx = std::max(mx, D.up_off[8 * l + oct + 1] - D.up_off[8 * l + oct]);
        dg::Args a{};
        a.A = D.m2m_oct; a.a_batch = (int64_t)nrep * nrep; a.lda = nrep; a.M = nrep; a.K = nrep;
        a.S = 1; a.nd = ND; a.X = D.up; a.ldx = nrep; a.in = D.up_child + u0; a.Y = D.tmpB; a.ldy = nrep;
        a.alpha = 1.0; a.add = 0; a.boff = D.up_off_dev + 8 * l;
        LB_DG(dg::gemm_cols(a, mx * ND, 8, st));
        const int64_t p0 = D.up_par_off[l], p1 = D.up_par_off[l + 1];
        if (p1 > p0) {
          m2m_sum_kernel<<<(unsigned)((p1 - p0) * ND), 128, 0, st>>>(D.tmpB, D.up_child8 + 8 * p0, D.up_par + p0,
                                                                     p1 - p0, ND, nrep, D.up);
          LB_CHECK_LAUNCH();
        }
      }
      continue;
    }
    for (int oct = 0; oct < 8; ++oct) {
      const int64_t g0 = D.up_off[8 * l + oct], g1 = D.up_off[8 * l + oct + 1];
      const int64_t cnt = g1 - g0;
      if (cnt == 0) continue;
      {
        grid_tensor_kernel<ND><<<(unsigned)cnt, 256, grid_smem, st>>>(
            D.up_child + g0, D.up_parent + g0, D.btgt_oct, D.m2m, n, D.up, D.up, 0);
      }
      LB_CHECK_LAUNCH();
    }
  }
  mark(2);
  // a sharded apply sums the ranks' partial upward expansions here (the hook
  // enqueues the all-reduce on this stream, lb_fmm_plan_set_upward_hook)
  if (P->up_hook) P->up_hook(P->up_hook_user, D.up, nb * ND * (int64_t)nrep, ND, (void*)st);
  // ---- M2L (fmm.py:873-886), by canonical key, chunked at target boundaries
  if (P->m2l_slices < 0) LB_TRY(ensure_lowrank(P, ND));
  else LB_TRY(ensure_oz(P, ND, st));
  // M2L: low-rank fused per key (default) or staged (the A/B probe switch)
  static const int m2l_mode = [] {  // LB_M2L_MODE=staged
    const char* e = std::getenv("LB_M2L_MODE");
    return (e && std::string(e) == "staged") ? 2 : 0;
  }();
  // fused mode: the first factor of every key and offset in ONE launch
  // (batches = lattice offsets, per-batch ranks), T of key k at tbase1[k] nd
  const bool lowrank_fused = P->m2l_slices < 0 && m2l_mode != 2 && nrep <= m2lf::max_nrep() &&
                             ND <= m2lf::kMaxNd && D.lo_rmax <= 4 * m2lf::kMaxKS;
  if (lowrank_fused && D.lo_gbatch > 0) {
    m2l1::Args a{};
    const int64_t q0 = D.lo_gb0;
    a.A = D.lr_bp; a.a_off = D.lo_gaoff; a.m_b = D.lo_gm; a.K = nrep; a.nd = ND; a.X = D.up;
    a.in = D.lo_src + q0; a.alpha_q = D.lo_scale + q0; a.out = D.lo_tcol + q0; a.Y = D.lr_t;
    a.y_off = D.lo_gyoff; a.boff = D.lo_gboff; a.tiles = D.lo_tiles[ND];
    LB_DG(m2l1::launch(a, D.lo_ntiles[ND], D.lo_rmax, st));
  }
  if (lowrank_fused) {
    // low-rank, fused: Y = A_k T and the permuted accumulation per unit of
    // whole target groups, Y kept in shared memory (T from the launch above);
    // every batch of units in one launch, its groups' sums then added to the
    // check values in key order
    const std::vector<int64_t>& bo = D.lo_batch_off[ND];
    const std::vector<int64_t>& bg = D.lo_batch_grp[ND];
    const int lut_n = D.lo_aff ? D.lo_lut_n : 0;
    for (size_t bi = 0; bi + 1 < bo.size(); ++bi) {
      if (bo[bi + 1] == bo[bi]) continue;
      m2lf::Args f{};
      f.A = m2lf::use_ring(nrep, lut_n) ? D.lr_ap : nullptr;
      f.Arow = D.lr_a; f.nrep = nrep; f.nd = ND; f.T = D.lr_t;
      f.urec = D.lo_units[ND] + m2lf::kRec * bo[bi]; f.tpair = D.v_tgt_pair_off;
      f.voff = D.v_off_idx; f.perm = D.perm;
      f.aff = reinterpret_cast<const int4*>(D.lo_aff); f.coords = D.lo_coords; f.lut = D.lo_lut;
      f.lut_n = D.lo_lut_n;
      f.part = D.lo_part; f.g0 = bg[bi];
      f.carry = D.lo_carry; f.carry_flag = D.lo_carry_flag; f.carry_slots = D.lo_carry_slots;
      LB_DG(m2lf::launch(f, bo[bi + 1] - bo[bi], D.lo_rmax, st));
      LB_DG(m2lf::reduce(D.lo_rt_tgt, D.lo_rt_off, D.lo_rt_grp, D.lo_rt_n, bg[bi], bg[bi + 1], D.lo_part, ND,
                         nrep, D.dc, st));
    }
  }
  for (int k = 0; k < P->ncanon && !lowrank_fused; ++k) {
    const int64_t pb = D.v_key_pair_off[k], pe = D.v_key_pair_off[k + 1];
    if (pe == pb) continue;
    const std::vector<int64_t> tp(D.v_tpoff_host.begin() + D.v_key_tgt_off[k],
                                  D.v_tpoff_host.begin() + D.v_key_tgt_off[k + 1] + 1);
    int64_t ti = 0;
    const int64_t ntg = (int64_t)tp.size() - 1;
    while (ti < ntg) {
      int64_t tj = ti;
      while (tj < ntg && tp[tj + 1] - tp[ti] <= D.tmp_cols) ++tj;
      if (tj == ti) tj = ti + 1;  // a single target with more pairs than the cap cannot occur (<= 316 offsets)
      const int64_t p0 = tp[ti], np = tp[tj] - tp[ti];
      if (P->m2l_slices > 0) {
        // gather + slice straight into the int8 column pack, tcgen05 GEMM
        const oz::ColGather g{D.up, D.v_src, D.v_off_idx, D.v_scale, D.perm_inv, p0, ND};
        const cudaError_t e = oz::m2l_gemm(P->m2l_slices, D.oz_a + (int64_t)k * oz::pack_rows_bytes(nrep, D.oz_S),
                                           D.oz_rs + (int64_t)k * ceil_div(nrep, oz::kBM) * oz::kBM, g, nrep,
                                           np * ND, D.oz_b, D.oz_cs, D.tmpB, st);
        if (e != cudaSuccess) return fail(LB_ERR_CUDA, std::string("m2l tcgen05 gemm: ") + cudaGetErrorString(e));
      } else {
        // the gathered column: scale(pi) * up[src(pi), l, perm_inv[off(pi), p]]
        dg::Args a{};
        a.S = 1; a.nd = ND; a.X = D.up; a.ldx = nrep; a.in = D.v_src + p0;
        a.kperm = D.perm_inv; a.kp = D.v_off_idx + p0; a.alpha_q = D.v_scale + p0;
        a.alpha = 1.0; a.add = 0; a.nq = np;
        if (P->m2l_slices < 0) {  // K_k ~= A_k B_k: T = B_k X (r_k x cols), Y = A_k T
          const int r = P->lr_rank[k];
          const int64_t o = P->lr_off[k] * nrep;
          a.A = D.lr_b + o; a.lda = nrep; a.M = r; a.K = nrep; a.Y = D.lr_t; a.ldy = r;
          LB_DG(dg::gemm_cols(a, np * ND, 1, st));
          LB_TRY(gemm_contig(D.lr_a + o, r, nrep, r, D.lr_t, r, D.tmpB, nrep, np * ND, 1.0, st));
        } else {  // the dense canonical operator (the reference's arithmetic)
          a.A = D.canon + (int64_t)k * nrep * nrep; a.lda = nrep; a.M = nrep; a.K = nrep;
          a.Y = D.tmpB; a.ldy = nrep;
          LB_DG(dg::gemm_cols(a, np * ND, 1, st));
        }
      }
      m2l_accum_kernel<<<(unsigned)(tj - ti), 128, 0, st>>>(D.tmpB, D.v_tgts, D.v_tgt_pair_off,
                                                            D.v_off_idx, D.perm,
                                                            D.v_key_tgt_off[k] + ti, p0, ND, nrep, D.dc);
      LB_CHECK_LAUNCH();
      ti = tj;
    }
  }
  mark(3);
  // ---- X list (fmm.py:888-911)
  if (D.n_x > 0) {
    LB_TRY(launch_lattice<ND>((unsigned)D.n_x, st, D.x_boxes, D.x_off, D.x_leaves, 0, D.bctr, D.bhalf, D.bsrc,
                              D.spos, D.cs, D.vs, t.ns, (int)dm_chunk, D.pts, nrep,
                              surface ? P->dc_scale : 1.0, 0, D.dc, 1, 1));
  }
  mark(4);
  // ---- L2L (fmm.py:913-935)
  for (int l = 0; l < t.nlev; ++l) {
    const int64_t s0 = D.level_slot_off[l], s1 = D.level_slot_off[l + 1];
    if (surface) {  // local = h pinv_dn @ dcheck over the level's slots (fmm.py:920)
      const double hl = t.half / std::ldexp(1.0, l);
      if (D.level_loc[l]) {
        LB_TRY(gemm_contig(D.pinv_dn, nrep, nrep, nrep, D.dc + s0 * ND * nrep, nrep,
                           D.loc + s0 * ND * nrep, nrep, (s1 - s0) * ND, hl, st));
      } else if (s1 > s0) {  // no check values anywhere on this level: local = 0
        LB_CUDA(cudaMemsetAsync(D.loc + s0 * ND * nrep, 0, sizeof(double) * (s1 - s0) * ND * nrep, st));
      }
    }
    if (l + 1 >= t.nlev) break;
    if (surface) {
      // dcheck[c] += l2l[octant] @ local[parent] / h_c (fmm.py:931-935): the
      // eight octant groups of level l+1 are the eight batches of one launch
      const double hc = t.half / std::ldexp(1.0, l + 1);
      int64_t mx = 0;
      for (int oct = 0; oct < 8; ++oct)
        mx = std::max(mx, D.dn_off[8 * (l + 1) + oct + 1] - D.dn_off[8 * (l + 1) + oct]);
      if (mx > 0) {
        dg::Args a{};
        a.A = D.l2l_oct; a.a_batch = (int64_t)nrep * nrep; a.lda = nrep; a.M = nrep; a.K = nrep;
        const int64_t d0 = D.dn_off[8 * (l + 1)];
        a.S = 1; a.nd = ND; a.X = D.loc; a.ldx = nrep; a.in = D.dn_parent + d0; a.Y = D.dc; a.ldy = nrep;
        a.out = D.dn_child + d0; a.alpha = 1.0 / hc; a.add = 1; a.boff = D.dn_off_dev + 8 * (l + 1);
        LB_DG(dg::gemm_cols(a, mx * ND, 8, st));
      }
      continue;
    }
    for (int oct = 0; oct < 8; ++oct) {
      const int64_t g0 = D.dn_off[8 * (l + 1) + oct], g1 = D.dn_off[8 * (l + 1) + oct + 1];
      const int64_t cnt = g1 - g0;
      if (cnt == 0) continue;
      {
        grid_tensor_kernel<ND><<<(unsigned)cnt, 256, grid_smem, st>>>(
            D.dn_child + g0, D.dn_parent + g0, D.btgt_oct, D.m2m, n, D.loc, D.dc, 1);
      }
      LB_CHECK_LAUNCH();
    }
  }
  mark(5);
  // ---- leaf stage (fmm.py:937-988)
  LB_CUDA(cudaMemsetAsync(D.tout, 0, sizeof(double) * ND * t.nt * 10, st));
  if (proj_out) {
    if (t.nt > 0) {
      gather_rows3_kernel<<<(unsigned)ceil_div(t.nt, 256), 256, 0, st>>>(proj_nrm, D.tgt_sorted, t.nt, D.tnrm);
      LB_CHECK_LAUNCH();
    }
    if (t.ns > 0) {
      gather_rows3_kernel<<<(unsigned)ceil_div(t.ns, 256), 256, 0, st>>>(proj_snrm, D.src_sorted, t.ns, D.snrm);
      LB_CHECK_LAUNCH();
    }
    LB_CUDA(cudaMemsetAsync(D.tproj, 0, sizeof(double) * 3 * t.nt, st));
  }
  if (D.n_tleaf > 0) {
    if (!surface) {
      const size_t sm = l2t_smem(n, level);
      LB_CUDA(cudaFuncSetAttribute(l2t_grid_kernel<ND>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   (int)l2t_smem(16, 2)));
      l2t_grid_kernel<ND><<<(unsigned)D.n_tleaf, kL2tBT, sm, st>>>(D.t_leaves, D.bctr, D.bhalf,
                                                                  D.btgt, D.tpos, t.nt, n, D.vinv,
                                                                  D.loc, level, D.tout);
      LB_CHECK_LAUNCH();
    }
    mark(6);
    // partial slots of split leaves for this chunk's accumulator width
    {
      const int64_t na = proj_out ? 3 : (int64_t)ND * ncomp(level);
      const int64_t need = D.part_doubles * na;
      if (need > D.leaf_part_cap) {
        cudaFree(D.leaf_part);
        D.leaf_part = nullptr;
        LB_CUDA(cudaMalloc((void**)&D.leaf_part, sizeof(double) * std::max<int64_t>(need, 1)));
        D.leaf_part_cap = need;
      }
      // items[4i+3] holds the partial offset in units of (target slots); scale
      // it to doubles for this width once per width change
      if (D.part_width != na) {
        scale_item_offsets_kernel<<<(unsigned)ceil_div(std::max<int64_t>(D.n_items, 1), 256), 256, 0, st>>>(
            D.leaf_items, D.leaf_item_slot, D.n_items, na);
        LB_CHECK_LAUNCH();
        D.part_width = na;
      }
    }
#define LB_LEAF(HD, LV)                                                                        \
  leaf_kernel<ND, HD, LV><<<(unsigned)D.n_items, kLeafBT, 0, st>>>(                                 \
      D.leaf_order, D.leaf_items, D.leaf_part,                                                  \
      D.t_leaves, D.u_off, D.u_list, D.w_off, D.w_list, D.bctr, D.bhalf, D.bsrc, D.btgt,       \
      D.spos, D.tpos, D.cs, D.vs, t.ns, t.nt, D.pts, nrep, surface ? 1 : 0, P->de_scale,      \
      surface ? P->ue_scale : 1.0, D.loc, D.up, D.tout);                                      \
  LB_CHECK_LAUNCH();                                                                           \
  if (D.n_split > 0)                                                                           \
    leaf_reduce_kernel<ND, ncomp(LV), false><<<(unsigned)D.n_split, 128, 0, st>>>(             \
        D.split_leaf, D.split_item_off, D.leaf_items, D.t_leaves, D.btgt, D.leaf_part, t.nt, D.tout)
    if constexpr (ND == 2) {
      if (proj_out) {  // projected leaf (fmm_apply_a3proj): writes tproj, not tout
        leaf_kernel<2, true, 2, true><<<(unsigned)D.n_items, kLeafBT, 0, st>>>(
            D.leaf_order, D.leaf_items, D.leaf_part,
            D.t_leaves, D.u_off, D.u_list, D.w_off, D.w_list, D.bctr, D.bhalf, D.bsrc, D.btgt,
            D.spos, D.tpos, D.cs, D.vs, t.ns, t.nt, D.pts, nrep, surface ? 1 : 0, P->de_scale,
            surface ? P->ue_scale : 1.0, D.loc, D.up, D.tproj, D.tnrm, D.snrm);
        LB_CHECK_LAUNCH();
        if (D.n_split > 0)
          leaf_reduce_kernel<2, 1, true><<<(unsigned)D.n_split, 128, 0, st>>>(
              D.split_leaf, D.split_item_off, D.leaf_items, D.t_leaves, D.btgt, D.leaf_part, t.nt, D.tproj);
        LB_CHECK_LAUNCH();
      }
    }
    if (proj_out) {
    } else if (hd) {
      if (level == 0) { LB_LEAF(true, 0); } else if (level == 1) { LB_LEAF(true, 1); } else { LB_LEAF(true, 2); }
    } else {
      if (level == 0) { LB_LEAF(false, 0); } else if (level == 1) { LB_LEAF(false, 1); } else { LB_LEAF(false, 2); }
    }
#undef LB_LEAF
    LB_CHECK_LAUNCH();
  }
  if (D.n_tleaf == 0) mark(6);
  mark(7);
  fmm_scatter_kernel<<<(unsigned)ceil_div((int64_t)ND * t.nt, 256), 256, 0, st>>>(
      D.tout, D.tgt_sorted, t.nt, ND, d0, level, pot, grad, hess);
  LB_CHECK_LAUNCH();
  if (proj_out && t.nt > 0) {
    scatter_proj_kernel<<<(unsigned)ceil_div(t.nt, 256), 256, 0, st>>>(D.tproj, D.tgt_sorted, t.nt, proj_out);
    LB_CHECK_LAUNCH();
  }
  mark(8);
  return LB_OK;
}

}  // namespace

void fmm_release_device(lb_fmm_plan* P) {
  FmmDevice& D = P->dev;
  void* ptrs[] = {D.spos, D.tpos, D.src_sorted, D.tgt_sorted, D.bctr, D.bhalf, D.bsrc, D.btgt,
                  D.pts, D.pinv_up, D.pinv_dn, D.m2m, D.l2l, D.canon, D.perm, D.perm_inv, D.vinv,
                  D.p2m_leaves, D.up_child, D.up_parent, D.dn_child, D.dn_parent, D.v_src,
                  D.v_tgt_pair_off, D.v_tgts, D.v_off_idx, D.v_scale, D.x_boxes, D.x_off,
                  D.x_leaves, D.t_leaves, D.u_off, D.u_list, D.w_off, D.w_list, D.cs, D.vs, D.up,
                  D.dc, D.tmpA, D.tmpB, D.tout, D.btgt_oct, D.tnrm, D.tproj, D.snrm,
                  D.leaf_items, D.leaf_item_slot, D.split_leaf, D.split_item_off, D.leaf_part, D.leaf_order};
  for (void* p : ptrs) cudaFree(p);
  if (P->rep == 0) cudaFree(D.loc);
  cudaFree(D.oz_a);
  cudaFree(D.oz_rs);
  cudaFree(D.lr_a);
  cudaFree(D.lr_b);
  cudaFree(D.lr_t);
  cudaFree(D.lo_carry);
  cudaFree(D.lo_carry_flag);
  cudaFree(D.lo_aff); cudaFree(D.lo_coords); cudaFree(D.lo_lut);
  cudaFree(D.lo_keytab); cudaFree(D.lo_rt_tgt); cudaFree(D.lo_rt_off); cudaFree(D.lo_rt_grp); cudaFree(D.lo_part);
  for (int i = 0; i < 5; ++i) cudaFree(D.lo_unit_key[i]);
  cudaFree(D.lr_ap);
  cudaFree(D.lr_bp); cudaFree(D.lo_src); cudaFree(D.lo_tcol); cudaFree(D.lo_scale);
  cudaFree(D.lo_boff); cudaFree(D.lo_aoff);
  cudaFree(D.lo_gboff); cudaFree(D.lo_gaoff); cudaFree(D.lo_gyoff); cudaFree(D.lo_gm);
  for (int i = 0; i < 5; ++i) {
    cudaFree(D.lo_units[i]);
    cudaFree(D.lo_tiles[i]);
  }
  cudaFree(D.oz_b);
  cudaFree(D.oz_cs);
  cudaFree(D.dn_off_dev);
  cudaFree(D.up_off_dev);
  cudaFree(D.src_own); cudaFree(D.cs_own); cudaFree(D.vs_own);
  cudaFree(D.up_par);
  cudaFree(D.up_child8);
  cudaFree(D.m2m_oct);
  cudaFree(D.l2l_oct);
  D = FmmDevice();
}

}  // namespace lb

using namespace lb;

extern "C" {

int lb_fmm_plan_set_operators(lb_fmm_plan* P, const lb_fmm_ops* o) {
  if (!P || !o) return fail(LB_ERR_ARG, "lb_fmm_plan_set_operators: null argument");
  if (o->rep != 0 && o->rep != 1) return fail(LB_ERR_ARG, "lb_fmm_plan_set_operators: rep must be 0 or 1");
  if (o->rep == 1 && (o->m < 2 || o->m > 16)) return fail(LB_ERR_ARG, "grid order must be in [2, 16]");
  const int nrep = o->nrep;
  const int64_t nn = (int64_t)nrep * nrep;
  fmm_release_device(P);
  P->rep = o->rep;
  P->m = o->m;
  P->nrep = nrep;
  P->pts.assign(o->pts, o->pts + 3 * nrep);
  if (o->rep == 0) {
    P->pinv_up.assign(o->pinv_up, o->pinv_up + nn);
    P->pinv_dn.assign(o->pinv_dn, o->pinv_dn + nn);
    P->m2m.assign(o->m2m, o->m2m + 8 * nn);
    P->l2l.assign(o->l2l, o->l2l + 8 * nn);
  } else {
    P->m2m.assign(o->m2m, o->m2m + 2 * o->m * o->m);
    P->vinv.assign(o->vinv, o->vinv + o->m * o->m);
  }
  P->ncanon = o->ncanon;
  P->canon.assign(o->canon, o->canon + (int64_t)o->ncanon * nn);
  P->noff = o->noff;
  P->off_vec.assign(o->off_vec, o->off_vec + 3 * o->noff);
  P->off_key.assign(o->off_key, o->off_key + o->noff);
  P->off_perm.assign(o->off_perm, o->off_perm + (int64_t)o->noff * nrep);
  return LB_OK;
}

int lb_fmm_plan_set_m2l_factors(lb_fmm_plan* P, const int32_t* ranks, const double* a, const double* b) {
  if (!P || !ranks || !a || !b) return fail(LB_ERR_ARG, "lb_fmm_plan_set_m2l_factors: null argument");
  if (P->ncanon <= 0 || P->nrep <= 0) return fail(LB_ERR_ARG, "lb_fmm_plan_set_m2l_factors: operators not set");
  std::vector<int64_t> off(P->ncanon + 1, 0);
  for (int k = 0; k < P->ncanon; ++k) {
    if (ranks[k] < 1 || ranks[k] > P->nrep)
      return fail(LB_ERR_ARG, "lb_fmm_plan_set_m2l_factors: rank outside [1, nrep]");
    off[k + 1] = off[k] + ranks[k];
  }
  P->lr_rank.assign(ranks, ranks + P->ncanon);
  P->lr_off = off;
  const size_t total = (size_t)off.back() * P->nrep;
  P->lr_a_host.assign(a, a + total);
  P->lr_b_host.assign(b, b + total);
  FmmDevice& D = P->dev;  // device copies are rebuilt on the next apply
  cudaFree(D.lr_a);
  cudaFree(D.lr_b);
  cudaFree(D.lr_ap);
  D.lr_a = D.lr_b = D.lr_ap = nullptr;
  return LB_OK;
}

int lb_fmm_plan_set_m2l(lb_fmm_plan* P, int slices) {
  if (!P) return fail(LB_ERR_ARG, "null plan");
  if (slices == -1) {
    if (P->lr_rank.empty()) return fail(LB_ERR_ARG, "lb_fmm_plan_set_m2l: low-rank M2L needs factors");
    P->m2l_slices = -1;
    return LB_OK;
  }
  if (slices != 0 && (slices < 3 || slices > 8))
    return fail(LB_ERR_ARG, "lb_fmm_plan_set_m2l: slices must be -1 (low rank), 0 (fp64) or in [3, 8]");
  if (slices != 0 && P->nrep > 2048)
    return fail(LB_ERR_ARG, "lb_fmm_plan_set_m2l: tensor-core M2L needs nrep <= 2048");
  P->m2l_slices = slices;
  return LB_OK;
}

int lb_fmm_plan_set_target_range(lb_fmm_plan* P, int64_t t0, int64_t t1) {
  if (!P) return fail(LB_ERR_ARG, "null plan");
  if (t1 >= 0 && (t0 < 0 || t0 > t1 || t1 > P->tree.nt))
    return fail(LB_ERR_SHAPE, "lb_fmm_plan_set_target_range: range outside [0, nt]");
  if (t0 == P->own_t0 && t1 == P->own_t1) return LB_OK;
  P->own_t0 = t0;
  P->own_t1 = t1;
  fmm_release_device(P);  // lists are rebuilt on the next apply
  return LB_OK;
}

int lb_fmm_plan_set_xw(lb_fmm_plan* P, int direct) {
  if (!P) return fail(LB_ERR_ARG, "null plan");
  if (direct != 0 && direct != 1) return fail(LB_ERR_ARG, "lb_fmm_plan_set_xw: mode must be 0 or 1");
  if (direct == P->xw_direct) return LB_OK;
  P->xw_direct = direct;
  fmm_release_device(P);  // the U / W / X device lists are rebuilt on the next apply
  return LB_OK;
}

int lb_fmm_plan_set_source_range(lb_fmm_plan* P, int64_t s0, int64_t s1) {
  if (!P) return fail(LB_ERR_ARG, "null plan");
  if (s1 >= 0 && (s0 < 0 || s0 > s1 || s1 > P->tree.ns))
    return fail(LB_ERR_SHAPE, "lb_fmm_plan_set_source_range: range outside [0, ns]");
  if (s0 == P->own_s0 && s1 == P->own_s1) return LB_OK;
  P->own_s0 = s0;
  P->own_s1 = s1;
  fmm_release_device(P);  // P2M / M2M lists are rebuilt on the next apply
  return LB_OK;
}

int lb_fmm_plan_set_upward_hook(lb_fmm_plan* P, lb_fmm_upward_hook hook, void* user) {
  if (!P) return fail(LB_ERR_ARG, "null plan");
  P->up_hook = hook;
  P->up_hook_user = user;
  return LB_OK;
}

int lb_fmm_plan_set_timing(lb_fmm_plan* P, int on) {
  if (!P) return fail(LB_ERR_ARG, "null plan");
  P->timing = on != 0;
  return LB_OK;
}

int lb_fmm_stage_times(const lb_fmm_plan* P, double* ms) {
  if (!P || !ms) return fail(LB_ERR_ARG, "null argument");
  for (int i = 0; i <= kStages; ++i) ms[i] = i < (int)P->stage_ms.size() ? P->stage_ms[i] : 0.0;
  return LB_OK;
}

}  // extern "C"

namespace lb {
int fmm_apply_impl(lb_fmm_plan* P, const double* charges, const double* dipoles, int nd,
                   uint32_t cmask, uint32_t dmask, int level, double* pot, double* grad,
                   double* hess, cudaStream_t st, const double* proj_nrm, double* proj_out,
                   const double* proj_snrm) {
  if (!P) return fail(LB_ERR_ARG, "lb_fmm_apply: null plan");
  if (P->rep < 0) return fail(LB_ERR_ARG, "lb_fmm_apply: operators not set");
  if (nd <= 0 || nd > 32) return fail(LB_ERR_SHAPE, "lb_fmm_apply: nd must be in [1, 32]");
  if (level < 0 || level > 2) return fail(LB_ERR_ARG, "lb_fmm_apply: level must be 0, 1 or 2");
  if (!pot || (level >= 1 && !grad) || (level >= 2 && !hess))
    return fail(LB_ERR_ARG, "lb_fmm_apply: missing output buffer");
  const uint32_t valid = nd == 32 ? 0xffffffffu : ((1u << nd) - 1u);
  cmask &= valid;
  dmask &= valid;
  if ((cmask && !charges) || (dmask && !dipoles))
    return fail(LB_ERR_ARG, "lb_fmm_apply: active mask without a density array");
  if (proj_out && (nd != 2 || level != 2 || !proj_nrm || !proj_snrm))
    return fail(LB_ERR_ARG, "fmm_apply_a3proj: two densities at level 2 with target and source normals");
  {
    const cudaError_t stale = cudaGetLastError();
    if (stale != cudaSuccess)
      return fail(LB_ERR_CUDA, std::string("lb_fmm_apply: error pending before the call: ") +
                                   cudaGetErrorString(stale));
  }
  if (!P->dev.ready) {
    const auto c0 = std::chrono::steady_clock::now();
    LB_TRY(build_device(P));
    P->setup_ms[3] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - c0).count();
  }
  if (proj_out && !P->dev.tproj) {
    const int64_t nt = std::max<int64_t>(P->tree.nt, 1);
    LB_CUDA(cudaMalloc((void**)&P->dev.tnrm, sizeof(double) * 3 * nt));
    LB_CUDA(cudaMalloc((void**)&P->dev.tproj, sizeof(double) * 3 * nt));
    LB_CUDA(cudaMalloc((void**)&P->dev.snrm, sizeof(double) * 3 * std::max<int64_t>(P->tree.ns, 1)));
  }
  std::vector<cudaEvent_t> ev;
  if (P->timing) {
    ev.resize(kStages + 1);
    for (auto& e : ev) cudaEventCreate(&e);
  }
  std::vector<double> acc(kStages + 1, 0.0);
  for (int d0 = 0; d0 < nd; d0 += 4) {
    const int ndc = std::min(4, nd - d0);
    LB_TRY(ensure_work(P, ndc));
    int rc;
    switch (ndc) {
      case 1: rc = apply_chunk<1>(P, d0, cmask, dmask, charges, dipoles, level, pot, grad, hess, st, ev); break;
      case 2:
        rc = apply_chunk<2>(P, d0, cmask, dmask, charges, dipoles, level, pot, grad, hess, st, ev,
                            proj_nrm, proj_out, proj_snrm);
        break;
      case 3: rc = apply_chunk<3>(P, d0, cmask, dmask, charges, dipoles, level, pot, grad, hess, st, ev); break;
      default: rc = apply_chunk<4>(P, d0, cmask, dmask, charges, dipoles, level, pot, grad, hess, st, ev); break;
    }
    if (rc != LB_OK) return rc;
    if (P->timing) {
      cudaEventSynchronize(ev[kStages]);
      float t = 0;
      for (int i = 0; i < kStages; ++i) {
        cudaEventElapsedTime(&t, ev[i], ev[i + 1]);
        acc[i] += t;
      }
      cudaEventElapsedTime(&t, ev[0], ev[kStages]);
      acc[kStages] += t;
    }
  }
  if (P->timing) {
    P->stage_ms = acc;
    for (auto& e : ev) cudaEventDestroy(e);
  }
  return LB_OK;
}

int fmm_apply_a3proj(lb_fmm_plan* P, const double* charges, const double* dipoles,
                     const double* tnrm, const double* snrm, double* pot, double* grad, double* hess,
                     double* proj, cudaStream_t st) {
  if (!proj) return fail(LB_ERR_ARG, "fmm_apply_a3proj: null projection output");
  return fmm_apply_impl(P, charges, dipoles, 2, 3u, 1u, 2, pot, grad, hess, st, tnrm, proj, snrm);
}
}  // namespace lb

extern "C" {

int lb_fmm_apply(lb_fmm_plan* P, const double* charges, const double* dipoles, int nd,
                 uint32_t cmask, uint32_t dmask, int level, double* pot, double* grad,
                 double* hess, void* stream) {
  return lb::fmm_apply_impl(P, charges, dipoles, nd, cmask, dmask, level, pot, grad, hess,
                            as_stream(stream), nullptr, nullptr, nullptr);
}

}  // extern "C"
