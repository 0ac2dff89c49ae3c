// Low-rank M2L, second half, fused with the permuted accumulation
// (fmm.py:873-886).  For one canonical key k with K_k ~= A_k B_k, the first
// factor T = B_k P_o x / h (rank x columns) comes from dgemm_cols.cuh (the
// permuted multipoles gathered straight into shared memory); this kernel
// takes a unit of whole target groups (pairs sorted by target), forms
//   Y = A_k T            (nrep x <= 32 columns, DMMA 8x8x4, in shared memory)
// and adds, per target and density, the pairs' Y read through the forward
// cube-symmetry permutation in their fixed order:
//   dc[t, l, i] += sum_{pairs of t} Y[perm[o, i], (pair, l)]
// so Y never leaves the SM (the staged path wrote and re-read 2 x 8 nrep
// bytes per pair and density).  A target group with more columns than one
// pass holds is done in consecutive passes of the same CTA (deterministic).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dgemm_cols.cuh"

namespace lb {
namespace m2lf {

constexpr int kThreads = 512;  // 16 warps: the accumulation is latency-bound
constexpr int kCols = 32;
constexpr int kMaxKS = 28;   // rank <= 112
constexpr int kMaxNd = 4;    // densities per FMM chunk
constexpr int kMaxIt = 2;    // nrep <= 2 * kThreads

struct Args {
  const double* A;           // A_k (nrep x r) row-major, lda = r
  int nrep, r, nd;
  const double* T;           // T column c of the chunk at T + c * r
  const int64_t* units;      // per unit: [first target group, end) (absolute group indices)
  const int64_t* vtgts;      // per target group: target slot
  const int64_t* tpair;      // per target group: first pair (absolute); tpair[g + 1] = end
  const int32_t* voff;       // per pair: offset index
  const int32_t* perm;       // (noff x nrep) forward permutations
  int64_t p0;                // absolute pair of T column 0 (the chunk's first pair)
  double* dc;                // (nbox, nd, nrep)
};

__host__ __device__ inline int ldy(int nrep) { return ((nrep + 7) / 8) * 8 + 1; }
inline size_t smem_bytes(int nrep) {
  return sizeof(double) * ((size_t)kCols * ldy(nrep) + (size_t)kCols * (((kMaxKS * 4 + 15) / 16) * 16 + 4));
}

__global__ void __launch_bounds__(kThreads, 1) m2l_fused_kernel(Args g) {  // <= 128 registers
  extern __shared__ __align__(16) double sm[];
  const int LY = ldy(g.nrep);
  double* Ys = sm;                          // [column][row], stride LY
  double* Ts = sm + (size_t)kCols * LY;     // [column][k], stride LT
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  const int64_t u = blockIdx.x;
  const int64_t tg0 = g.units[2 * u], tg1 = g.units[2 * u + 1];
  const int64_t pa = g.tpair[tg0], pe = g.tpair[tg1];
  const int64_t total = (pe - pa) * g.nd;
  const int KS = (g.r + 3) / 4;
  const int LT = ((KS * 4 + 15) / 16) * 16 + 4;  // Ts column stride
  const int mtiles = (g.nrep + 7) / 8;
  double carry[kMaxNd][kMaxIt];  // a multi-pass group's per-thread sums
#pragma unroll
  for (int l = 0; l < kMaxNd; ++l)
#pragma unroll
    for (int j = 0; j < kMaxIt; ++j) carry[l][j] = 0.0;
  for (int64_t cb = 0; cb < total; cb += kCols) {
    const int ncol = (int)min((int64_t)kCols, total - cb);
    __syncthreads();  // the previous pass's accumulation is done with Ys
    // T columns of this pass, zero-padded to 4 * KS rows and 32 columns;
    // consecutive threads read consecutive k of one column (coalesced) and
    // store it column-major, Ts[c][k] at stride LT (LT = 4 mod 16 doubles:
    // conflict-free fragment reads, as in dgemm_cols.cuh)
    for (int e = tid; e < KS * 4 * kCols; e += kThreads) {
      const int c = e / (KS * 4), k = e % (KS * 4);
      const int64_t col = (pa - g.p0) * g.nd + cb + c;
      Ts[c * LT + k] = (c < ncol && k < g.r) ? g.T[col * g.r + k] : 0.0;
    }
    __syncthreads();
    // Y = A_k T: warp w takes M-tiles w, w + 16, ...; all four N-tiles; the
    // A_k fragments stream from L2 eight k-steps at a time
    for (int mt = warp; mt < mtiles; mt += kThreads / 32) {
      const int row = mt * 8 + gq;
      double acc[4][2];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) acc[nt][0] = acc[nt][1] = 0.0;
      for (int k0 = 0; k0 < KS; k0 += 8) {
        double a[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          const int k = (k0 + j) * 4 + tq;
          a[j] = (k0 + j < KS && row < g.nrep && k < g.r) ? __ldg(g.A + (int64_t)row * g.r + k) : 0.0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (k0 + j >= KS) break;
          const double* tp = Ts + gq * LT + (k0 + j) * 4 + tq;
#pragma unroll
          for (int nt = 0; nt < 4; ++nt) dg::dmma(acc[nt][0], acc[nt][1], a[j], tp[nt * 8 * LT]);
        }
      }
      // D[row = mt*8 + gq][col = nt*8 + 2 tq + h]
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) {
        const int c = nt * 8 + 2 * tq;
        Ys[(size_t)c * LY + mt * 8 + gq] = acc[nt][0];
        Ys[(size_t)(c + 1) * LY + mt * 8 + gq] = acc[nt][1];
      }
    }
    __syncthreads();
    // per target group and density, pairs in order, through the permutation.
    // A unit is whole target groups of <= kCols columns, or ONE larger group
    // done in passes: its sums carry over the passes in registers, so every
    // target's sum runs over its pairs in the same order whatever nd is
    // (a density's result does not depend on the other densities)
    if (tg1 - tg0 == 1 && total > kCols) {
      const int64_t tb = g.vtgts[tg0];
#pragma unroll
      for (int l = 0; l < kMaxNd; ++l) {
        if (l >= g.nd) break;
#pragma unroll
        for (int j = 0; j < kMaxIt; ++j) {
          const int i = tid + j * kThreads;
          if (i >= g.nrep) break;
          double acc = carry[l][j];
          for (int c = l - (int)(cb % g.nd); c < ncol; c += g.nd) {
            if (c < 0) continue;
            const int64_t q = pa + (cb + c) / g.nd;
            acc += Ys[(size_t)c * LY + g.perm[(int64_t)g.voff[q] * g.nrep + i]];
          }
          carry[l][j] = acc;
        }
      }
      if (cb + kCols >= total) {
#pragma unroll
        for (int l = 0; l < kMaxNd; ++l) {
          if (l >= g.nd) break;
#pragma unroll
          for (int j = 0; j < kMaxIt; ++j) {
            const int i = tid + j * kThreads;
            if (i < g.nrep) g.dc[(tb * g.nd + l) * (int64_t)g.nrep + i] += carry[l][j];
          }
        }
      }
      continue;
    }
    for (int64_t tg = tg0; tg < tg1; ++tg) {
      const int64_t q0 = g.tpair[tg], q1 = g.tpair[tg + 1];
      const int64_t tb = g.vtgts[tg];
      for (int l = 0; l < g.nd; ++l) {
        double* d = g.dc + (tb * g.nd + l) * (int64_t)g.nrep;
        for (int i = tid; i < g.nrep; i += kThreads) {
          double acc = 0.0;
          for (int64_t q = q0; q < q1; ++q)
            acc += Ys[(size_t)((q - pa) * g.nd + l - cb) * LY + g.perm[(int64_t)g.voff[q] * g.nrep + i]];
          d[i] += acc;
        }
      }
    }
  }
}

inline cudaError_t launch(const Args& a, int64_t nunits, cudaStream_t st) {
  if (nunits <= 0) return cudaSuccess;
  if (a.r > 4 * kMaxKS || a.nd > kMaxNd || a.nrep > kMaxIt * kThreads) return cudaErrorInvalidValue;
  static int attr = 0;
  const int need = (int)smem_bytes(a.nrep);
  if (need > attr) {
    const cudaError_t e = cudaFuncSetAttribute(m2l_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, need);
    if (e != cudaSuccess) return e;
    attr = need;
  }
  m2l_fused_kernel<<<(unsigned)nunits, kThreads, need, st>>>(a);
  return cudaGetLastError();
}

}  // namespace m2lf
}  // namespace lb
