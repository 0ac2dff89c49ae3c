// Low-rank M2L, first half (fmm.py:873-886): for every lattice offset d of
// every canonical key k (K_k ~= A_k B_k), the thin product
//   T[:, c] = (1 / h) (B_k P_d) x[src(c)]      (r_k x columns of offset d)
// on the FP64 tensor cores (DMMA 8x8x4), all offsets of all keys in ONE
// launch over a flat tile list.  The shape that matters is the thin M = r_k
// (30 - 80 at the precisions in use, different for every key): the generic
// gather-GEMM (dgemm_cols.cuh) pads M to its 64-row tile and spent 43% of its
// tensor-pipe time on padding at BASELINE config 3 (ncu, profiles/round2:
// 61% pipe-active for 35% useful).  Here a CTA owns ALL rows of its batch in
// 8-row M-tiles (ceil(r_k / 8) of them, nothing padded past the last tile),
// 128 columns; of its 16 warps eight take the first half of the M-tiles and
// eight the second, 16 columns each (8 warps per CTA left the tensor pipe at
// 62%: two warps per scheduler do not cover the DMMA issue latency), so a warp
// runs about ceil(r_k / 16) x 2 independent DMMA chains per 4-deep k-step.  K (= nrep) streams in chunks of 32 through a
// three-stage cp.async pipeline; k-steps past K are skipped, not zero-padded.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#include "dgemm_cols.cuh"

namespace lb {
namespace m2l1 {

constexpr int kBN = 128;
constexpr int kThreads = 512;  // 16 warps: 2 (halves of the M-tiles) x 8 (16 columns each)
constexpr int kStages = 3;
constexpr int kMaxMT = 14;  // rank <= 112 (m2l_fused.cuh: kMaxKS * 4)

struct Args {
  const double* A;           // batch z: (B_k P_d) row-major (m_b[z] x K) at A + a_off[z], lda = K
  const int64_t* a_off;
  const int32_t* m_b;        // rows (rank) of batch z
  int K, nd;
  const double* X;           // upward expansions: column (b, l) at X + (b * nd + l) * K
  const int64_t* in;         // per pair q: source box slot
  const double* alpha_q;     // per pair q: 1 / h
  const int64_t* out;        // per pair q: T column of the pair within its key
  double* Y;                 // T: batch z's key at Y + y_off[z] * nd, column stride m_b[z] rounded up to 4
                             // (m2lf::tstride; the pad rows stay zero from the allocation)
  const int64_t* y_off;
  const int64_t* boff;       // batch z holds pairs [boff[z], boff[z + 1]) - boff[0]
  const int32_t* tiles;      // per CTA: (batch, first column / kBN)
};

template <int MT>
struct Smem {
  static constexpr int kRows = MT * 8;
  static constexpr size_t kBytes = sizeof(double) * kStages * (size_t)(kRows + kBN) * dg::kLD;
};

// The CTA's whole tile for a batch of NMT 8-row M-tiles (compile-time, so the
// DMMAs of absent M-tiles do not exist: predicated-off DMMAs still occupy the
// tensor pipe, ncu profiles/round2).
template <int NMT>
__device__ __forceinline__ void run_tile(const Args& g, double* dsm, const double* const* xin,
                                         double* const* yout, const double* alph, const double* A,
                                         int Mz) {
  constexpr int R = NMT * 8;
  auto As = [&](int b) { return dsm + (size_t)b * (R + kBN) * dg::kLD; };
  auto Xs = [&](int b) { return dsm + (size_t)b * (R + kBN) * dg::kLD + (size_t)R * dg::kLD; };
  const int K = g.K;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int gq = lane >> 2, tq = lane & 3;
  // 16-byte copies need even K (row / column strides) and aligned bases
  const bool v16 = (K & 1) == 0 && (((uintptr_t)A | (uintptr_t)g.X) & 15) == 0;

  // warps 0-7 take the first H M-tiles, warps 8-15 the rest; 16 columns each
  constexpr int H = (NMT + 1) / 2;
  const int wm = warp >> 3, wn = warp & 7;
  double acc[H][2][2];
#pragma unroll
  for (int i = 0; i < H; ++i)
#pragma unroll
    for (int j = 0; j < 2; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  const int nchunk = (K + dg::kKC - 1) / dg::kKC;
  auto load = [&](int buf, int k0) {
    double* as = As(buf);
    double* xs = Xs(buf);
    if (v16) {
      for (int e = tid; e < R * (dg::kKC / 2); e += kThreads) {
        const int rr = e / (dg::kKC / 2), kk = (e % (dg::kKC / 2)) * 2, k = k0 + kk;
        int bytes = 0;
        if (rr < Mz && k < K) bytes = (k + 1 < K) ? 16 : 8;
        dg::cp16(as + rr * dg::kLD + kk, bytes ? A + (int64_t)rr * K + k : g.A, bytes);
      }
      for (int e = tid; e < kBN * (dg::kKC / 2); e += kThreads) {
        const int c = e / (dg::kKC / 2), kk = (e % (dg::kKC / 2)) * 2, k = k0 + kk;
        const double* base = xin[c];
        int bytes = 0;
        if (base && k < K) bytes = (k + 1 < K) ? 16 : 8;
        dg::cp16(xs + c * dg::kLD + kk, bytes ? base + k : g.X, bytes);
      }
    } else {
      for (int e = tid; e < R * dg::kKC; e += kThreads) {
        const int rr = e / dg::kKC, kk = e % dg::kKC, k = k0 + kk;
        const bool ok = rr < Mz && k < K;
        dg::cp8(as + rr * dg::kLD + kk, ok ? A + (int64_t)rr * K + k : g.A, ok);
      }
      for (int e = tid; e < kBN * dg::kKC; e += kThreads) {
        const int c = e >> 5, kk = e & 31, k = k0 + kk;
        const double* base = xin[c];
        const bool ok = base != nullptr && k < K;
        dg::cp8(xs + c * dg::kLD + kk, ok ? base + k : g.X, ok);
      }
    }
  };
  // one K chunk of this warp's NM M-tiles (compile-time NM)
  auto chunk = [&](auto nm_c, const double* as, const double* xs, int ksn) {
    constexpr int NM = decltype(nm_c)::value;
#pragma unroll
    for (int ks = 0; ks < dg::kKC / 4; ++ks) {
      if (ks >= ksn) break;
      const int kk = ks * 4 + tq;
      const double b0 = xs[kk], b1 = xs[8 * dg::kLD + kk];
      double a[NM > 0 ? NM : 1];
#pragma unroll
      for (int mt = 0; mt < NM; ++mt) a[mt] = as[mt * 8 * dg::kLD + kk];
#pragma unroll
      for (int mt = 0; mt < NM; ++mt) {
        dg::dmma(acc[mt][0][0], acc[mt][0][1], a[mt], b0);
        dg::dmma(acc[mt][1][0], acc[mt][1][1], a[mt], b1);
      }
    }
  };

  // prologue: kStages - 1 chunks in flight (empty groups keep the count uniform)
#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (s < nchunk) load(s, s * dg::kKC);
    dg::cp_commit();
  }
  for (int i = 0; i < nchunk; ++i) {
    dg::cp_wait<kStages - 2>();  // chunk i has landed
    __syncthreads();             // ... for every thread; chunk i - 1's buffer is free
    if (i + kStages - 1 < nchunk) load((i + kStages - 1) % kStages, (i + kStages - 1) * dg::kKC);
    dg::cp_commit();
    const int buf = i % kStages;
    const double* as = As(buf) + (wm * H * 8 + gq) * dg::kLD;
    const double* xs = Xs(buf) + (wn * 16 + gq) * dg::kLD;
    const int ksn = min(dg::kKC / 4, (K - i * dg::kKC + 3) / 4);  // k-steps with any k < K
    if (wm == 0) chunk(std::integral_constant<int, H>{}, as, xs, ksn);
    else chunk(std::integral_constant<int, NMT - H>{}, as, xs, ksn);
  }
  // epilogue: D[row = mt*8 + gq][col = wn*16 + nt*8 + 2 tq + h], scaled by 1/h
  const int nm_w = wm == 0 ? H : NMT - H;
#pragma unroll
  for (int mt = 0; mt < H; ++mt) {
    const int row = (wm * H + mt) * 8 + gq;
    if (mt >= nm_w || row >= Mz) continue;
#pragma unroll
    for (int nt = 0; nt < 2; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn * 16 + nt * 8 + 2 * tq + h;
        double* y = yout[c];
        if (y) y[row] = alph[c] * acc[mt][nt][h];
      }
    }
  }
}

template <int MT>
__global__ void __launch_bounds__(kThreads, 1) first_kernel(Args g) {
  extern __shared__ __align__(16) double dsm[];
  __shared__ const double* xin[kBN];
  __shared__ double* yout[kBN];
  __shared__ double alph[kBN];

  const int z = g.tiles[2 * blockIdx.x];
  const int64_t c0 = (int64_t)g.tiles[2 * blockIdx.x + 1] * kBN;
  const int64_t q0 = g.boff[z] - g.boff[0], q1 = g.boff[z + 1] - g.boff[0];
  const int64_t ncols = (q1 - q0) * g.nd;
  const int Mz = g.m_b[z];
  const int nmt = (Mz + 7) / 8;
  const double* A = g.A + g.a_off[z];
  double* const Yz = g.Y + g.y_off[z] * g.nd;
  const int tid = threadIdx.x;

  for (int j = tid; j < kBN; j += kThreads) {
    const int64_t c = c0 + j;
    const bool ok = c < ncols;
    const int64_t q = q0 + (ok ? c / g.nd : 0);
    const int l = ok ? (int)(c % g.nd) : 0;
    xin[j] = ok ? g.X + (g.in[q] * g.nd + l) * (int64_t)g.K : nullptr;
    yout[j] = ok ? Yz + (g.out[q] * g.nd + l) * (int64_t)(((Mz + 3) / 4) * 4) : nullptr;
    alph[j] = ok ? g.alpha_q[q] : 0.0;
  }
  __syncthreads();
#define LB_M2L1_CASE(N)                                          \
  case N:                                                        \
    if constexpr (N <= MT) run_tile<N>(g, dsm, xin, yout, alph, A, Mz); \
    break;
  switch (nmt) {
    LB_M2L1_CASE(1) LB_M2L1_CASE(2) LB_M2L1_CASE(3) LB_M2L1_CASE(4) LB_M2L1_CASE(5)
    LB_M2L1_CASE(6) LB_M2L1_CASE(7) LB_M2L1_CASE(8) LB_M2L1_CASE(9) LB_M2L1_CASE(10)
    LB_M2L1_CASE(11) LB_M2L1_CASE(12) LB_M2L1_CASE(13) LB_M2L1_CASE(14)
    default: break;
  }
#undef LB_M2L1_CASE
}

template <int MT>
inline cudaError_t launch_mt(const Args& a, int64_t ntiles, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(first_kernel<MT>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)Smem<MT>::kBytes);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  first_kernel<MT><<<(unsigned)ntiles, kThreads, Smem<MT>::kBytes, st>>>(a);
  return cudaGetLastError();
}

// rmax: the largest rank of any batch
inline cudaError_t launch(const Args& a, int64_t ntiles, int rmax, cudaStream_t st) {
  if (ntiles <= 0) return cudaSuccess;
  if (rmax > 8 * kMaxMT || a.nd < 1) return cudaErrorInvalidValue;
  if (rmax <= 64) return launch_mt<8>(a, ntiles, st);
  if (rmax <= 80) return launch_mt<10>(a, ntiles, st);
  return launch_mt<kMaxMT>(a, ntiles, st);
}

}  // namespace m2l1
}  // namespace lb
