// Low-rank M2L, second half, fused with the permuted accumulation
// (fmm.py:873-886).  For one canonical key k with K_k ~= A_k B_k, the first
// factor T = B_k P_o x / h (rank x columns) comes from m2l_first.cuh; this
// kernel takes a unit of whole target groups of ONE key (pairs sorted by key,
// then target), forms
//   Y = A_k T            (nrep x <= 16 columns, DMMA 8x8x4, in shared memory)
// and adds, per target and density, the pairs' Y read through the forward
// cube-symmetry permutation in their fixed order:
//   dc[t, l, i] += sum_{pairs of t} Y[perm[o, i], (pair, l)]
// so Y never leaves the SM (the staged path wrote and re-read 2 x 8 nrep
// bytes per pair and density).  One launch per key: a (target, key) group
// belongs to exactly one unit, so within a launch no two CTAs touch the same
// dc entry and the += is a plain read-modify-write; the keys' launches are
// stream-ordered, which fixes the order of every target's sums.
//
// A pass holds kCols / nd whole pairs (a pair's nd columns never straddle two
// passes).  A target group with more pairs than one pass is the only group of
// its unit and runs in consecutive passes of the same CTA, its running sums
// parked in a scratch slot between passes (claimed from a small global pool),
// so every target's sum runs over its pairs in the same order whatever nd is.
//
// Shape (ncu, profiles/round2): the three phases of a unit -- T tile in, the
// tensor-core product, the latency-bound permuted accumulation -- serialise
// inside a CTA, so the tile is sized for TWO CTAs per SM (16 columns, 8
// warps, <= 128 registers): one CTA's DMMAs run under the other's
// accumulation.  In the product a warp holds up to four 8-row M-tiles x two
// N-tiles in registers: per 4-deep k-step four A_k fragment loads (from L2,
// through a per-warp cp.async ring, L1 bypassed, one k-step pair ahead), two T
// fragment loads (shared memory) and eight DMMAs.  M- and N-tile counts are compile-time in every
// instantiation: a predicated-off DMMA still occupies the tensor pipe.  The
// accumulation reads each pair's permutation index once for all its densities
// with four pairs in flight; the dc rows a unit updates are prefetched into
// L1 before the product.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "dgemm_cols.cuh"

namespace lb {
namespace m2lf {

constexpr int kThreads = 256;  // 8 warps
constexpr int kWarps = kThreads / 32;
constexpr int kCols = 16;
constexpr int kNT = kCols / 8;
constexpr int kMaxKS = 28;   // rank <= 112
constexpr int kMaxNd = 4;    // densities per FMM chunk
constexpr int kMW = 4;       // M-tiles a warp holds at once

// columns one pass holds for nd densities (whole pairs)
__host__ __device__ inline int pass_cols(int nd) { return (kCols / nd) * nd; }

struct Args {
  const double* A;           // A_k in fragment order (pack_a), or nullptr: no ring, use Arow
  const double* Arow;        // A_k (nrep x r) row-major, lda = r
  int nrep, r, nd;
  const double* T;           // T column c of the key at T + c * tstride(r), rows >= r zero
  const int64_t* units;      // per unit: [first target group, end) (absolute group indices)
  const int64_t* vtgts;      // per target group: target slot
  const int64_t* tpair;      // per target group: first pair (absolute); tpair[g + 1] = end
  const int32_t* voff;       // per pair: offset index
  const int32_t* perm;       // (noff x nrep) forward permutations
  int64_t p0;                // absolute pair of T column 0 (the key's first pair)
  double* dc;                // (nbox, nd, nrep)
  double* carry;             // multi-pass groups: pool of carry_slots x (kMaxNd * nrep) doubles
  unsigned* carry_flag;      // per slot: 0 free, 1 taken (zero-initialised)
  int carry_slots;
};

// T's column stride in global memory: whole 4-deep k-steps (32-byte columns)
__host__ __device__ inline int tstride(int r) { return ((r + 3) / 4) * 4; }
__host__ __device__ inline int ldy(int nrep) { return ((nrep + 7) / 8) * 8 + 1; }
__host__ __device__ constexpr int ldt() { return ((kMaxKS * 4 + 15) / 16) * 16 + 4; }

__device__ __forceinline__ void prefetch_l1(const void* p) {
  asm volatile("prefetch.global.L1 [%0];\n" ::"l"(p));
}

// A_k in DMMA fragment order (pack_a below): per M-tile mt and k-step PAIR
// kp, 32 lanes x 2 doubles -- lane (gq, tq) holds A[mt*8 + gq][(2 kp + h)*4 + tq],
// h = 0, 1 -- zero past nrep rows / r columns.  A warp's fetch of one (mt, kp)
// is one coalesced 512-byte cp.async.cg (L2 -> shared, L1 bypassed); every
// lane reads back only the 16 bytes it copied, so the ring needs no barrier,
// only cp.async.wait_group.
__host__ __device__ inline int kpairs(int r) { return (((r + 3) / 4) + 1) / 2; }
inline size_t packed_doubles(int nrep, int r) { return (size_t)((nrep + 7) / 8) * kpairs(r) * 64; }
inline void pack_a(const double* A, int nrep, int r, double* out) {
  const int mtiles = (nrep + 7) / 8, KP = kpairs(r);
  for (int mt = 0; mt < mtiles; ++mt)
    for (int kp = 0; kp < KP; ++kp)
      for (int lane = 0; lane < 32; ++lane)
        for (int h = 0; h < 2; ++h) {
          const int row = mt * 8 + (lane >> 2), k = (2 * kp + h) * 4 + (lane & 3);
          out[(((size_t)mt * KP + kp) * 32 + lane) * 2 + h] = (row < nrep && k < r) ? A[(size_t)row * r + k] : 0.0;
        }
}

constexpr int kRing = 2;  // k-step pairs in flight per warp
constexpr size_t kRingDoubles = (size_t)kWarps * kRing * kMW * 32 * 2;

// Y = A_k T for one pass, one round of a warp's M-tiles: NM M-tiles (mt0,
// mt0 + kWarps, ...) x NTN N-tiles in registers; the A_k fragments arrive
// through the warp's cp.async ring one k-step pair (2 NM NTN DMMAs) ahead.
template <int NTN, int NM>
__device__ __forceinline__ void gemm_round(const double* __restrict__ Ap, int r, int mt0,
                                           const double* Ts, double* Ys, int LY, double* ring) {
  constexpr int LT = ldt();
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int KS = (r + 3) / 4, KP = (KS + 1) / 2;
  const double* src[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) src[m] = Ap + ((size_t)(mt0 + m * kWarps) * KP * 32 + lane) * 2;
  double* const rg = ring + lane * 2;  // [stage][m][lane][2]
  double acc[NM][NTN][2];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) acc[m][nt][0] = acc[m][nt][1] = 0.0;
  const double* tp = Ts + gq * LT + tq;
  auto issue = [&](int kp) {
    if (kp < KP) {
#pragma unroll
      for (int m = 0; m < NM; ++m) dg::cp16(rg + ((kp & 1) * kMW + m) * 64, src[m] + (size_t)kp * 64, 16);
    }
    dg::cp_commit();
  };
  issue(0);
  for (int kp = 0; kp < KP; ++kp) {
    issue(kp + 1);
    dg::cp_wait<1>();  // pair kp has landed (this lane's own 16 bytes)
    double2 a[NM];
#pragma unroll
    for (int m = 0; m < NM; ++m) a[m] = *reinterpret_cast<const double2*>(rg + ((kp & 1) * kMW + m) * 64);
    {
      double b[NTN];
#pragma unroll
      for (int nt = 0; nt < NTN; ++nt) b[nt] = tp[nt * 8 * LT + kp * 8];
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int nt = 0; nt < NTN; ++nt) dg::dmma(acc[m][nt][0], acc[m][nt][1], a[m].x, b[nt]);
    }
    if (2 * kp + 1 < KS) {
      double b[NTN];
#pragma unroll
      for (int nt = 0; nt < NTN; ++nt) b[nt] = tp[nt * 8 * LT + kp * 8 + 4];
#pragma unroll
      for (int m = 0; m < NM; ++m)
#pragma unroll
        for (int nt = 0; nt < NTN; ++nt) dg::dmma(acc[m][nt][0], acc[m][nt][1], a[m].y, b[nt]);
    }
  }
  dg::cp_wait<0>();
  // D[row = mt*8 + gq][col = nt*8 + 2 tq + h]
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int row = (mt0 + m * kWarps) * 8 + gq;
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) {
      const int c = nt * 8 + 2 * tq;
      Ys[(size_t)c * LY + row] = acc[m][nt][0];
      Ys[(size_t)(c + 1) * LY + row] = acc[m][nt][1];
    }
  }
}

// The same round with the A_k fragments loaded straight from the row-major
// A_k (L2, L1 bypassed) into registers one k-step ahead: no ring, for the
// expansion sizes whose Y tile leaves no shared memory for one at two CTAs
// per SM (the grid representations, nrep >= 729).  Rows past nrep in the last
// M-tile are clamped to the last row (computed, stored into Ys' padding rows,
// never read).
__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];\n" : "=d"(v) : "l"(p));
  return v;
}
template <int NTN, int NM>
__device__ __forceinline__ void gemm_round_ldg(const double* __restrict__ A, int r, int nrep, int mt0,
                                               const double* Ts, double* Ys, int LY) {
  constexpr int LT = ldt();
  const int lane = threadIdx.x & 31;
  const int gq = lane >> 2, tq = lane & 3;
  const int KS = (r + 3) / 4;
  const double* ap[NM];
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int row = min((mt0 + m * kWarps) * 8 + gq, nrep - 1);
    ap[m] = A + (int64_t)row * r + tq;
  }
  double acc[NM][NTN][2];
#pragma unroll
  for (int m = 0; m < NM; ++m)
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) acc[m][nt][0] = acc[m][nt][1] = 0.0;
  const double* tp = Ts + gq * LT + tq;
  auto load_a = [&](int ks, double (&a)[NM]) {
    const bool ok = ks * 4 + tq < r;
#pragma unroll
    for (int m = 0; m < NM; ++m) a[m] = ok ? ld_stream(ap[m] + ks * 4) : 0.0;
  };
  auto step = [&](int ks, const double (&a)[NM]) {
    double b[NTN];
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) b[nt] = tp[nt * 8 * LT + ks * 4];
#pragma unroll
    for (int m = 0; m < NM; ++m)
#pragma unroll
      for (int nt = 0; nt < NTN; ++nt) dg::dmma(acc[m][nt][0], acc[m][nt][1], a[m], b[nt]);
  };
  double a0[NM], a1[NM];
  load_a(0, a0);
  for (int ks = 0; ks < KS; ks += 2) {
    if (ks + 1 < KS) load_a(ks + 1, a1);
    step(ks, a0);
    if (ks + 1 < KS) {
      if (ks + 2 < KS) load_a(ks + 2, a0);
      step(ks + 1, a1);
    }
  }
#pragma unroll
  for (int m = 0; m < NM; ++m) {
    const int row = (mt0 + m * kWarps) * 8 + gq;
#pragma unroll
    for (int nt = 0; nt < NTN; ++nt) {
      const int c = nt * 8 + 2 * tq;
      Ys[(size_t)c * LY + row] = acc[m][nt][0];
      Ys[(size_t)(c + 1) * LY + row] = acc[m][nt][1];
    }
  }
}

// all rounds of this warp: M-tiles warp, warp + kWarps, ... in groups of kMW
template <int NTN, bool RING>
__device__ __forceinline__ void gemm_phase(const double* __restrict__ Ap, const double* __restrict__ Arow,
                                           int r, int nrep, const double* Ts, double* Ys, int LY,
                                           double* ring_base) {
  const int warp = threadIdx.x >> 5;
  const int mtiles = (nrep + 7) / 8;
  double* const ring = ring_base + (size_t)warp * kRing * kMW * 64;
  for (int mt0 = warp; mt0 < mtiles; mt0 += kMW * kWarps) {
    const int nm = min(kMW, (mtiles - mt0 + kWarps - 1) / kWarps);
    if constexpr (!RING) {
      switch (nm) {
        case 1: gemm_round_ldg<NTN, 1>(Arow, r, nrep, mt0, Ts, Ys, LY); break;
        case 2: gemm_round_ldg<NTN, 2>(Arow, r, nrep, mt0, Ts, Ys, LY); break;
        case 3: gemm_round_ldg<NTN, 3>(Arow, r, nrep, mt0, Ts, Ys, LY); break;
        default: gemm_round_ldg<NTN, 4>(Arow, r, nrep, mt0, Ts, Ys, LY); break;
      }
      continue;
    }
    switch (nm) {
      case 1: gemm_round<NTN, 1>(Ap, r, mt0, Ts, Ys, LY, ring); break;
      case 2: gemm_round<NTN, 2>(Ap, r, mt0, Ts, Ys, LY, ring); break;
      case 3: gemm_round<NTN, 3>(Ap, r, mt0, Ts, Ys, LY, ring); break;
      default: gemm_round<NTN, 4>(Ap, r, mt0, Ts, Ys, LY, ring); break;
    }
  }
}

template <bool RING>
__global__ void __launch_bounds__(kThreads, 2) m2l_fused_kernel(Args g) {  // <= 128 registers
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_poff[kCols];         // perm row offset (offset index x nrep) of the pass's pairs
  __shared__ int64_t s_gq[kCols + 1];   // first pair of the unit's groups (one-pass units)
  __shared__ int64_t s_gt[kCols];       // their target slots
  __shared__ int s_slot;                // a multi-pass unit's carry slot
  constexpr int LT = ldt();
  const int nd = g.nd, nrep = g.nrep, r = g.r;
  const int LY = ldy(nrep);
  double* Ys = sm;                          // [column][row], stride LY
  double* Ts = sm + (size_t)kCols * LY;     // [column][k], stride LT
  const int tid = threadIdx.x;
  const int64_t u = blockIdx.x;
  const int64_t tg0 = g.units[2 * u], tg1 = g.units[2 * u + 1];
  const int ngrp = (int)(tg1 - tg0);
  const int64_t pa = g.tpair[tg0], pe = g.tpair[tg1];
  const int ppp = kCols / nd;  // pairs per pass
  const bool multi = (pe - pa) > ppp;  // one group in several passes
  const int K4 = tstride(r);

  // group table (a multi-pass unit has one group)
  for (int e = tid; e <= ngrp && e <= kCols; e += kThreads) s_gq[e] = g.tpair[tg0 + e];
  for (int e = tid; e < ngrp && e < kCols; e += kThreads) s_gt[e] = g.vtgts[tg0 + e];
  if (multi && tid == 0) {  // claim a carry slot (the pool outnumbers the resident CTAs)
    unsigned s = (unsigned)((u * 2654435761ull) % (unsigned)g.carry_slots);
    while (atomicCAS(g.carry_flag + s, 0u, 1u) != 0u) s = (s + 1) % (unsigned)g.carry_slots;
    s_slot = (int)s;
  }
  __syncthreads();
  // the dc rows this unit updates, towards L1 while the product runs
  for (int e = 0; e < ngrp && e < kCols; ++e) {
    const double* d = g.dc + s_gt[e] * nd * (int64_t)nrep;
    for (int i = tid * 4; i < nd * nrep; i += kThreads * 4) prefetch_l1(d + i);
  }
  double* const carry = multi ? g.carry + (size_t)s_slot * kMaxNd * nrep : nullptr;

  for (int64_t pb = pa; pb < pe; pb += ppp) {
    const int np = (int)min((int64_t)ppp, pe - pb);
    const int ncol = np * nd;
    const int ntn = (ncol + 7) / 8;  // N-tiles in use
    __syncthreads();  // the previous pass's accumulation is done with Ys / s_poff
    // T columns of this pass (global columns are tstride(r) doubles, zero past
    // r): 16-byte cp.async copies into Ts[c][k] at stride LT (LT = 4 mod 16
    // doubles: conflict-free fragment reads, as in dgemm_cols.cuh); the
    // columns past ncol of the last N-tile are zeroed
    {
      const int h4 = K4 / 2;  // 16-byte pieces per column
      const double* Tc = g.T + (pb - g.p0) * nd * (int64_t)K4;
      for (int e = tid; e < h4 * ntn * 8; e += kThreads) {
        const int c = e / h4, k = (e - c * h4) * 2;
        dg::cp16(Ts + c * LT + k, c < ncol ? Tc + (int64_t)c * K4 + k : g.T, c < ncol ? 16 : 0);
      }
      dg::cp_commit();
      if (tid < np) s_poff[tid] = g.voff[pb + tid] * nrep;
      dg::cp_wait<0>();
    }
    __syncthreads();
    if (ntn == 1) gemm_phase<1, RING>(g.A, g.Arow, r, nrep, Ts, Ys, LY, Ts + (size_t)kCols * LT);
    else gemm_phase<kNT, RING>(g.A, g.Arow, r, nrep, Ts, Ys, LY, Ts + (size_t)kCols * LT);
    __syncthreads();
    // per target group and density, pairs in order, through the permutation:
    // one index per (pair, row) for all densities, four pairs in flight
    for (int e = 0; e < (multi ? 1 : ngrp); ++e) {
      const int64_t q0 = multi ? pa : s_gq[e], q1 = multi ? pe : s_gq[e + 1];
      const int ja = (int)(max(q0, pb) - pb), jb = (int)(min(q1, pb + np) - pb);
      if (ja >= jb) continue;
      const bool first = (pb + ja) == q0, last = (pb + jb) == q1;
      double* const d0 = g.dc + s_gt[e] * nd * (int64_t)nrep;
      for (int i = tid; i < nrep; i += kThreads) {
        double s[kMaxNd], old[kMaxNd];
#pragma unroll
        for (int l = 0; l < kMaxNd; ++l) {
          s[l] = (first || l >= nd) ? 0.0 : carry[(size_t)l * nrep + i];
          old[l] = (last && l < nd) ? d0[(int64_t)l * nrep + i] : 0.0;
        }
        const int32_t* pi = g.perm + i;
        for (int jp = ja; jp < jb; jp += 4) {
          int id[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) id[v] = (jp + v < jb) ? pi[s_poff[jp + v]] : 0;
#pragma unroll
          for (int v = 0; v < 4; ++v) {
            if (jp + v >= jb) break;
            const double* y = Ys + (size_t)((jp + v) * nd) * LY + id[v];
#pragma unroll
            for (int l = 0; l < kMaxNd; ++l)
              if (l < nd) s[l] += y[(size_t)l * LY];
          }
        }
#pragma unroll
        for (int l = 0; l < kMaxNd; ++l) {
          if (l >= nd) break;
          if (last) d0[(int64_t)l * nrep + i] = old[l] + s[l];
          else carry[(size_t)l * nrep + i] = s[l];
        }
      }
    }
  }
  if (multi) {  // hand the carry slot back
    __syncthreads();
    if (tid == 0) {
      __threadfence();
      atomicExch(g.carry_flag + s_slot, 0u);
    }
  }
}

inline size_t smem_bytes(int nrep, bool ring) {
  return sizeof(double) * ((size_t)kCols * ldy(nrep) + (size_t)kCols * ldt() + (ring ? kRingDoubles : 0));
}
// the ring variant when two CTAs with a ring fit one SM (227 KB, 1 KB reserved per CTA)
inline bool use_ring(int nrep) { return 2 * (smem_bytes(nrep, true) + 1024 + 512) <= 227 * 1024; }

// slots of the carry pool: four per SM (two CTAs are resident per SM)
inline int carry_slots(int sm_count) { return 4 * sm_count; }

// largest nrep one CTA's tile fits in shared memory for
inline int max_nrep() { return (int)((226 * 1024 / sizeof(double) - (size_t)kCols * ldt()) / kCols) - 8; }

inline cudaError_t launch(const Args& a, int64_t nunits, cudaStream_t st) {
  if (nunits <= 0) return cudaSuccess;
  if (a.r > 4 * kMaxKS || a.nd > kMaxNd || a.nd < 1 || !a.carry || !a.carry_flag || a.carry_slots < 1 ||
      a.nrep > max_nrep())
    return cudaErrorInvalidValue;
  if ((a.A == nullptr) == use_ring(a.nrep) || !a.Arow) return cudaErrorInvalidValue;
  const bool ring = a.A != nullptr;
  const int need = (int)smem_bytes(a.nrep, ring);
  static int attr[2] = {0, 0};
  if (need > attr[ring]) {
    const cudaError_t e = ring ? cudaFuncSetAttribute(m2l_fused_kernel<true>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, need)
                               : cudaFuncSetAttribute(m2l_fused_kernel<false>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, need);
    if (e != cudaSuccess) return e;
    attr[ring] = need;
  }
  if (ring) m2l_fused_kernel<true><<<(unsigned)nunits, kThreads, need, st>>>(a);
  else m2l_fused_kernel<false><<<(unsigned)nunits, kThreads, need, st>>>(a);
  return cudaGetLastError();
}

}  // namespace m2lf
}  // namespace lb
