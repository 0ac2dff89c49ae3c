// FP64 "gather - GEMM - scatter" on the FP64 tensor cores (DMMA 8x8x4,
// mma.sync.m8n8k4.f64), the one GEMM shape every FMM translation has:
//
//   Y[:, out(c)] (=|+=) alpha(c) * sum_{s < S} A_s * X[perm_c(:), in_s(c)]
//
// A_s row-major (M x K, lda), X / Y column vectors of an expansion array
// (one vector of K (X) or M (Y) doubles per (box, density)).  Logical column
// c = q * nd + l walks the launch's box / pair list q and the densities l.
// Per column the input vector of segment s is X + (in[s](q) * nd + l) * ldx
// (in == nullptr: q itself; an index of -1 skips that segment for the
// column), optionally read through a K-permutation (kperm + kp(q) * K: the
// M2L's cube-symmetry gather), and the output is Y + (out(q) * nd + l) * ldy.
// Batches (blockIdx.z) select A_z = A + z * a_batch and the box range
// [boff[z] - boff[0], boff[z+1] - boff[0]) (the M2M / L2L per-octant child
// groups).
//
// Every FMM stage maps onto it (fmm.py:823-935): P2M (pinv_up), M2M (the
// children of one level in 8 octant batches, then an in-order sum into the
// parents), L2L (pinv_dn, then l2l[octant] in 8 batches) and the M2L (its
// low-rank factors, or the dense canonical operators).
//
// Tiles: BM x BN per CTA, warps of WM x 32 (WM/8 M-tiles x 4 N-tiles of 8x8,
// WM/8 * 4 DMMAs per 4-deep k-step).  K runs in chunks of KC through an
// NS-stage cp.async ring with one block barrier per chunk (A rows 16-byte
// coalesced when aligned, X 16 B per contiguous pair or 8 B per gathered
// element, zero-filled past K); fragments come from shared memory at a
// (KC + 4)-double stride (two wavefronts per 8-byte fragment load, the
// minimum for 32 x 8 B).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace lb {
namespace dg {

constexpr int kKC = 32;      // K chunk and smem row stride (doubles) of m2l_first.cuh's tiles
constexpr int kLD = 36;
constexpr int kMaxSeg = 8;

struct Args {
  const double* A;           // segment s of batch z at A + z*a_batch + s*a_seg
  int64_t a_batch, a_seg;    // (or at A + a_off[z] + s*a_seg when a_off is set)
  const int64_t* a_off;
  int lda, M, K, S, nd;
  const double* X;           // input expansion array
  int64_t ldx;
  const int64_t* in;         // (nq_total x S) box index per segment, -1 = none; nullptr = q
  const int32_t* kperm;      // optional (nperm x K) K-permutations
  const int32_t* kp;         // per box/pair q: permutation index (with kperm)
  double* Y;
  int64_t ldy;
  const int64_t* out;        // per q output box; nullptr = q
  const double* alpha_q;     // optional per-q scale
  double alpha;
  int add;                   // 1: Y += ..., 0: Y = ...
  int64_t nq;                // boxes/pairs (no batches)
  const int64_t* boff;       // batches: q range [boff[z] - boff[0], boff[z+1] - boff[0])
  // optional per-batch shapes (the M2L's first factor over all keys at once):
  // rows m_b[z] (<= M), output at Y + y_off[z] * nd with column stride ldy_b[z]
  const int32_t* m_b;
  const int64_t* y_off;
  const int32_t* ldy_b;
};

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// src-size below the copy size zero-fills the rest (0: all zeros, src unread)
__device__ __forceinline__ void cp8(double* s, const double* g, bool valid) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(sa), "l"(g), "r"(valid ? 8 : 0));
}
__device__ __forceinline__ void cp16(double* s, const double* g, int bytes) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(s);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(sa), "l"(g), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int BM, int BN, int WM, int KC, int NS>
struct Cfg {
  static constexpr int kWarpsM = BM / WM, kWarpsN = BN / 32;
  static constexpr int kThreads = 32 * kWarpsM * kWarpsN;
  static constexpr int kMT = WM / 8;
  static constexpr int kLD = KC + 4;  // smem row stride (doubles)
  static constexpr size_t kSmem = sizeof(double) * NS * (BM + BN) * kLD;
};

template <int BM, int BN, int WM, int KC, int NS>
__global__ void __launch_bounds__(Cfg<BM, BN, WM, KC, NS>::kThreads) gemm_cols_kernel(Args g) {
  using C = Cfg<BM, BN, WM, KC, NS>;
  constexpr int NT = C::kThreads, MT = C::kMT;
  constexpr int kKC = KC, kLD = C::kLD;  // (shadow the namespace's m2l_first constants)
  static_assert(KC % 4 == 0 && NS >= 2, "K chunk in 4-deep k-steps, at least two stages");
  extern __shared__ __align__(16) double dsm[];
  // stage b: A tile at dsm + b * (BM + BN) * kLD, X tile BM * kLD behind it
  auto As = [&](int b) { return dsm + b * (BM + BN) * kLD; };
  auto Xs = [&](int b) { return dsm + b * (BM + BN) * kLD + BM * kLD; };
  __shared__ const double* xin[kMaxSeg][BN];
  __shared__ const int32_t* kpp[BN];
  __shared__ double* yout[BN];
  __shared__ double alph[BN];
  __shared__ int seg_used[kMaxSeg];
  __shared__ int x16;

  const int z = blockIdx.z;
  const int64_t q0 = g.boff ? g.boff[z] - g.boff[0] : 0;
  const int64_t q1 = g.boff ? g.boff[z + 1] - g.boff[0] : g.nq;
  const int64_t ncols = (q1 - q0) * g.nd;
  const int64_t c0 = (int64_t)blockIdx.y * BN;
  if (c0 >= ncols) return;
  const int m0 = blockIdx.x * BM;
  const int Mz = g.m_b ? g.m_b[z] : g.M;
  if (m0 >= Mz) return;
  const double* A = g.a_off ? g.A + g.a_off[z] : g.A + (int64_t)z * g.a_batch;
  double* const Yz = g.Y + (g.y_off ? g.y_off[z] * g.nd : 0);
  const int64_t ldyz = g.ldy_b ? g.ldy_b[z] : g.ldy;
  // 16-byte A copies need even row strides / offsets and an aligned base
  const bool a16 = ((g.lda | g.a_seg | g.a_batch) & 1) == 0 && (((uintptr_t)A) & 15) == 0;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp % C::kWarpsM, wn = warp / C::kWarpsM;
  const int gq = lane >> 2, tq = lane & 3;

  if (tid < kMaxSeg) seg_used[tid] = 0;
  if (tid == 0) x16 = (g.kperm == nullptr && (g.ldx & 1) == 0) ? 1 : 0;
  __syncthreads();
  for (int j = tid; j < BN; j += NT) {
    const int64_t c = c0 + j;
    const bool ok = c < ncols;
    const int64_t q = q0 + (ok ? c / g.nd : 0);
    const int l = ok ? (int)(c % g.nd) : 0;
    for (int s = 0; s < g.S; ++s) {
      const int64_t b = g.in ? g.in[q * g.S + s] : q;
      const double* p = (ok && b >= 0) ? g.X + (b * g.nd + l) * g.ldx : nullptr;
      xin[s][j] = p;
      if (p) {
        seg_used[s] = 1;  // benign race: every writer stores 1
        if (((uintptr_t)p) & 15) x16 = 0;
      }
    }
    kpp[j] = (ok && g.kperm) ? g.kperm + (int64_t)g.kp[q] * g.K : nullptr;
    const int64_t ob = g.out ? g.out[q] : q;
    yout[j] = ok ? Yz + (ob * g.nd + l) * ldyz : nullptr;
    alph[j] = ok ? g.alpha * (g.alpha_q ? g.alpha_q[q] : 1.0) : 0.0;
  }
  __syncthreads();
  const bool xv = x16 != 0;

  double acc[MT][4][2];
#pragma unroll
  for (int i = 0; i < MT; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // the (segment, chunk) sequence, skipping segments no column uses
  const int nchunk = (g.K + kKC - 1) / kKC;
  int nstep = 0;
  for (int s = 0; s < g.S; ++s) nstep += seg_used[s] ? nchunk : 0;
  auto step_at = [&](int i, int& s, int& k0) {
    for (s = 0; s < g.S; ++s) {
      if (!seg_used[s]) continue;
      if (i < nchunk) break;
      i -= nchunk;
    }
    k0 = i * kKC;
  };
  auto load = [&](int buf, int s, int k0) {
    const double* As_src = A + (int64_t)s * g.a_seg;
    double* as = As(buf);
    if (a16) {
      for (int e = tid; e < BM * (kKC / 2); e += NT) {
        const int r = e / (kKC / 2), kk = (e % (kKC / 2)) * 2;
        const int row = m0 + r, k = k0 + kk;
        int bytes = 0;
        if (row < Mz && k < g.K) bytes = (k + 1 < g.K) ? 16 : 8;
        cp16(as + r * kLD + kk, bytes ? As_src + (int64_t)row * g.lda + k : g.A, bytes);
      }
    } else {
      for (int e = tid; e < BM * kKC; e += NT) {
        const int r = e / kKC, kk = e % kKC;
        const int row = m0 + r, k = k0 + kk;
        const bool ok = row < Mz && k < g.K;
        cp8(as + r * kLD + kk, ok ? As_src + (int64_t)row * g.lda + k : g.A, ok);
      }
    }
    double* xs = Xs(buf);
    if (xv) {  // contiguous, 16-byte aligned columns
      for (int e = tid; e < BN * (kKC / 2); e += NT) {
        const int c = e / (kKC / 2), kk = (e % (kKC / 2)) * 2, k = k0 + kk;
        const double* base = xin[s][c];
        int bytes = 0;
        if (base && k < g.K) bytes = (k + 1 < g.K) ? 16 : 8;
        cp16(xs + c * kLD + kk, bytes ? base + k : g.X, bytes);
      }
    } else {
      for (int e = tid; e < BN * kKC; e += NT) {
        const int c = e / kKC, kk = e % kKC, k = k0 + kk;
        const double* base = xin[s][c];
        const bool ok = base != nullptr && k < g.K;
        const int32_t* pp = kpp[c];
        cp8(xs + c * kLD + kk, ok ? base + (pp ? pp[k] : k) : g.X, ok);
      }
    }
    cp_commit();
  };

  // ring: steps i .. i + NS - 2 in flight while step i is multiplied; one
  // commit group per step (empty past the end) keeps the wait count fixed
  for (int p = 0; p < NS - 1; ++p) {
    if (p < nstep) {
      int s, k0;
      step_at(p, s, k0);
      load(p, s, k0);
    } else {
      cp_commit();
    }
  }
  for (int i = 0; i < nstep; ++i) {
    const int buf = i % NS;
    cp_wait<NS - 2>();
    __syncthreads();  // step i has landed for every thread; buffer (i - 1) % NS is free
    if (i + NS - 1 < nstep) {
      int s, k0;
      step_at(i + NS - 1, s, k0);
      load((i + NS - 1) % NS, s, k0);
    } else {
      cp_commit();
    }
    const double* as = As(buf) + (wm * WM + gq) * kLD;
    const double* xs = Xs(buf) + (wn * 32 + gq) * kLD;
#pragma unroll
    for (int ks = 0; ks < kKC / 4; ++ks) {
      const int kk = ks * 4 + tq;
      double a[MT], b[4];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt) a[mt] = as[mt * 8 * kLD + kk];
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) b[nt] = xs[nt * 8 * kLD + kk];
#pragma unroll
      for (int mt = 0; mt < MT; ++mt)
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(acc[mt][nt][0], acc[mt][nt][1], a[mt], b[nt]);
    }
  }
  // epilogue: D[row][col] with row = gq, cols = 2 tq, 2 tq + 1 of each tile
#pragma unroll
  for (int mt = 0; mt < MT; ++mt) {
    const int row = m0 + wm * WM + mt * 8 + gq;
    if (row >= Mz) continue;
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int c = wn * 32 + nt * 8 + 2 * tq + h;
        double* y = yout[c];
        if (!y) continue;
        const double v = alph[c] * acc[mt][nt][h];
        y[row] = g.add ? y[row] + v : v;
      }
    }
  }
}

template <int BM, int BN, int WM, int KC = 32, int NS = 2>
inline cudaError_t launch(const Args& a, int64_t max_cols, int batches, cudaStream_t st) {
  using C = Cfg<BM, BN, WM, KC, NS>;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e = cudaFuncSetAttribute(gemm_cols_kernel<BM, BN, WM, KC, NS>,
                                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                                               (int)C::kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const dim3 grid((unsigned)((a.M + BM - 1) / BM), (unsigned)((max_cols + BN - 1) / BN),
                  (unsigned)batches);
  gemm_cols_kernel<BM, BN, WM, KC, NS><<<grid, C::kThreads, C::kSmem, st>>>(a);
  return cudaGetLastError();
}

// host launcher: grid = (M tiles, column tiles, batches).  The tile is the
// largest that still puts two CTAs' worth of work on every SM (148 SMs): the
// FMM's launches range from a few hundred columns (one level's parents, one
// offset's V pairs) to millions, and a small launch on big tiles leaves most
// SMs idle (measured: 48 CTAs for a config-3 M2L factor at 128 x 128)
inline cudaError_t gemm_cols(const Args& a, int64_t max_cols_per_batch, int batches, cudaStream_t st) {
  if (max_cols_per_batch <= 0 || batches <= 0 || a.M <= 0) return cudaSuccess;
  if (a.S < 1 || a.S > kMaxSeg) return cudaErrorInvalidValue;
  auto ctas = [&](int bm, int bn) {
    return (int64_t)((a.M + bm - 1) / bm) * ((max_cols_per_batch + bn - 1) / bn) * batches;
  };
  const int64_t want = 2 * 148;
  if (a.m_b) {  // per-batch row counts: 64-row tiles, the tiles past a batch's rows exit
    if (ctas(64, 128) >= want) return launch<64, 128, 32>(a, max_cols_per_batch, batches, st);
    return launch<64, 64, 32>(a, max_cols_per_batch, batches, st);
  }
  // Translation shapes (M > 64, K = M = nrep): the tile is chosen by a wave
  // model measured on a B200 at M = K = 488 (profiles/round2/
  // leaf_overlap_and_tiles.md).  A CTA's time is set by its own K loop
  // (DMMA latency x accumulators per warp, one barrier per chunk), not by
  // how many CTAs share the SM, so a launch costs (full waves) x tw + the
  // last wave (t1 if it fits one CTA per SM, else tw), in units that scale
  // with K alike for every tile: what matters is how the CTA count falls on
  // the 148 x occupancy slots.  The FMM's bottom levels are one to three
  // waves, where the best tile beats the old fixed choice by 20-30%.
  if (a.M > 64) {
    struct Cand { int id; int bm, bn; double t1, tw; int slots; };
    static const Cand cands[] = {{0, 64, 64, 39.0, 52.0, 296},
                                 {1, 64, 96, 60.0, 70.0, 296},
                                 {2, 64, 128, 60.0, 93.0, 296},
                                 {3, 128, 128, 93.0, 93.0, 148}};
    // a launch too small to put a 64 x 64 CTA on most SMs is bound by ONE
    // CTA's serial K loop: 32 x 32 tiles cut that loop's DMMA count four-fold
    if (ctas(64, 64) <= 100) return launch<32, 32, 16>(a, max_cols_per_batch, batches, st);
    int best = 0;
    double best_t = 1e300;
    for (const Cand& c : cands) {
      const int64_t n = ctas(c.bm, c.bn);
      const int64_t full = n / c.slots, rem = n % c.slots;
      const double t = full * c.tw + (rem == 0 ? 0.0 : (rem <= 148 ? c.t1 : c.tw));
      if (t < best_t - 1e-9) {
        best_t = t;
        best = c.id;
      }
    }
    switch (best) {
      case 0: return launch<64, 64, 32>(a, max_cols_per_batch, batches, st);
      case 1: return launch<64, 96, 32, 16, 4>(a, max_cols_per_batch, batches, st);
      case 2: return launch<64, 128, 32, 16, 3>(a, max_cols_per_batch, batches, st);
      default: return launch<128, 128, 32>(a, max_cols_per_batch, batches, st);
    }
  }
  if (a.M > 32) {
    if (ctas(64, 128) >= want) return launch<64, 128, 32>(a, max_cols_per_batch, batches, st);
    if (ctas(64, 64) >= 148) return launch<64, 64, 32>(a, max_cols_per_batch, batches, st);
    return launch<32, 32, 16>(a, max_cols_per_batch, batches, st);
  }
  if (ctas(32, 128) >= want) return launch<32, 128, 32>(a, max_cols_per_batch, batches, st);
  return launch<32, 64, 16>(a, max_cols_per_batch, batches, st);
}

}  // namespace dg
}  // namespace lb
