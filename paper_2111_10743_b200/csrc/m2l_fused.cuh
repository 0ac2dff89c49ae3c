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
// bytes per pair and density).  A (target, key) group belongs to exactly one
// unit and writes its sum, WRITE ONLY, to its own slot of a scratch buffer;
// reduce_kernel then adds every target's slots to its check values in key
// order.  So units of all keys run in ONE launch (heaviest ranks first; a
// batch of units when the slots would not fit the scratch buffer), no CTA
// waits on a read-modify-write of dc (the exposed L2 round trip per group was
// the accumulation's largest stall), there are no atomics, and every check
// value is the same left-to-right sum over the keys as a stream-ordered
// launch per key gave: bit-identical results.
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
// accumulation computes each pair's permuted row once for all its densities
// -- in closed form where the permutations are axis permutations and flips of
// the expansion lattice (fit_symmetries; three IMADs and a shared-memory
// table instead of a global index load), four pairs in flight.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <vector>

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
constexpr int kRec = 8;      // int64 per unit record

// columns one pass holds for nd densities (whole pairs)
__host__ __device__ inline int pass_cols(int nd) { return (kCols / nd) * nd; }

struct Args {
  const double* A;           // all keys' A_k in fragment order (pack_a), or nullptr: no ring, use Arow
  const double* Arow;        // all keys' A_k (nrep x r_k) row-major, lda = r_k
  int nrep, nd;
  const double* T;           // all keys' T (first factor)
  // per unit ONE 64-byte record, so a CTA's start is one dependent load deep
  // (key -> key table -> group range -> pair range was four: ncu showed 45% of
  // the grid-representation kernel's samples on those loads and the T tile's):
  // offset of its key's A_k in A and in Arow, offset of its first T column in
  // T, the key's rank, its first target group, its group count, its pair
  // range [pa, pe)
  const int64_t* urec;       // kRec int64 per unit
  const int64_t* tpair;      // per target group: first pair (absolute); tpair[g + 1] = end
  const int32_t* voff;       // per pair: offset index
  const int32_t* perm;       // (noff x nrep) forward permutations
  // the same permutations in closed form (fit_symmetries below; nullptr: use
  // the table): point i has lattice coordinates coords[i] = a | b << 8 | c << 16
  // on the m^3 lattice, offset d maps them to the lattice index
  // aff[d] = (A, B, C, D): A a + B b + C c + D, and lut turns that into the
  // expansion index
  const int4* aff;
  const uint32_t* coords;
  const uint16_t* lut;
  int lut_n;                 // m^3
  // every (target, key) group's sum goes to its own slot of `part`, write
  // only: slot = group index - g0, nd x nrep doubles (reduce_kernel adds the
  // slots into the check values in key order)
  double* part;
  int64_t g0;
  double* carry;             // multi-pass groups: pool of carry_slots x (kMaxNd * nrep) doubles
  unsigned* carry_flag;      // per slot: 0 free, 1 taken (zero-initialised)
  int carry_slots;
  int64_t nunits;            // units of this launch (set by launch(); urec holds that many records)
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

// One CTA per unit, no A_k ring: the kernel of the expansion sizes whose Y
// tile leaves no shared memory for a ring at two CTAs per SM (grid
// representations, nrep >= 729).  Kept beside the persistent kernel below
// because that one is slower here (10^6 points, eps 1e-9: M2L 66.3 ms with
// this kernel, 67.5-69.3 ms persistent, with or without cross-unit prefetch).
__global__ void __launch_bounds__(kThreads, 2) m2l_fused_unit_kernel(Args g) {  // <= 128 registers
  constexpr bool RING = false;
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_poff[kCols];         // perm row offset (offset index x nrep) of the pass's pairs
  __shared__ int4 s_aff[kCols];         // ... or their permutations in closed form
  __shared__ int64_t s_gq[kCols + 1];   // first pair of the unit's groups (one-pass units)
  __shared__ int s_slot;                // a multi-pass unit's carry slot
  constexpr int LT = ldt();
  const int nd = g.nd, nrep = g.nrep;
  const int LY = ldy(nrep);
  double* Ys = sm;                          // [column][row], stride LY
  double* Ts = sm + (size_t)kCols * LY;     // [column][k], stride LT
  const int tid = threadIdx.x;
  const int64_t u = blockIdx.x;
  const longlong2* const rp = reinterpret_cast<const longlong2*>(g.urec + kRec * u);
  const longlong2 r0 = __ldg(rp), r1 = __ldg(rp + 1), r2 = __ldg(rp + 2), r3 = __ldg(rp + 3);
  const double* const Ap = g.A ? g.A + r0.x : nullptr;
  const double* const Arow = g.Arow + r0.y;
  const double* const Tu = g.T + r1.x;  // the unit's first T column
  const int r = (int)r1.y;
  const int64_t tg0 = r2.x;
  const int ngrp = (int)r2.y;
  const int64_t pa = r3.x, pe = r3.y;
  const int ppp = kCols / nd;  // pairs per pass
  const bool multi = (pe - pa) > ppp;  // one group in several passes
  const int K4 = tstride(r);

  // T columns of a pass (global columns are tstride(r) doubles, zero past r):
  // 16-byte cp.async copies into Ts[c][k] at stride LT (LT = 4 mod 16 doubles:
  // conflict-free fragment reads, as in dgemm_cols.cuh); the columns past ncol
  // of the last N-tile are zeroed.  The first pass's copies are issued before
  // anything else so that they fly under the rest of the CTA's set-up.
  auto issue_T = [&](int64_t pb) {
    const int ncol = (int)min((int64_t)ppp, pe - pb) * nd;
    const int ntn = (ncol + 7) / 8;
    const int h4 = K4 / 2;  // 16-byte pieces per column
    const double* Tc = Tu + (pb - pa) * nd * (int64_t)K4;
    for (int e = tid; e < h4 * ntn * 8; e += kThreads) {
      const int c = e / h4, k = (e - c * h4) * 2;
      dg::cp16(Ts + c * LT + k, c < ncol ? Tc + (int64_t)c * K4 + k : g.T, c < ncol ? 16 : 0);
    }
    dg::cp_commit();
  };
  issue_T(pa);
  // lattice index -> expansion index, behind the tiles (and the ring)
  uint16_t* const s_lut = reinterpret_cast<uint16_t*>(Ts + (size_t)kCols * LT + (RING ? kRingDoubles : 0));
  if (g.aff)
    for (int e = tid; e < g.lut_n; e += kThreads) s_lut[e] = g.lut[e];
  // group table (a multi-pass unit has one group)
  for (int e = tid; e <= ngrp && e <= kCols; e += kThreads) s_gq[e] = g.tpair[tg0 + e];
  if (multi && tid == 0) {  // claim a carry slot (the pool outnumbers the resident CTAs)
    unsigned s = (unsigned)((u * 2654435761ull) % (unsigned)g.carry_slots);
    while (atomicCAS(g.carry_flag + s, 0u, 1u) != 0u) s = (s + 1) % (unsigned)g.carry_slots;
    s_slot = (int)s;
  }
  __syncthreads();
  double* const carry = multi ? g.carry + (size_t)s_slot * kMaxNd * nrep : nullptr;

  for (int64_t pb = pa; pb < pe; pb += ppp) {
    const int np = (int)min((int64_t)ppp, pe - pb);
    const int ncol = np * nd;
    const int ntn = (ncol + 7) / 8;  // N-tiles in use
    if (pb != pa) {
      __syncthreads();  // the previous pass's accumulation is done with Ys / s_poff
      issue_T(pb);
    }
    // the pairs' offsets (and their closed-form permutations: a dependent
    // load) are only needed by the accumulation: loaded here, parked in
    // registers under the product, stored after it -- the barrier before the
    // product does not wait for them
    int pd = 0;
    int4 paf = make_int4(0, 0, 0, 0);
    if (tid < np) pd = g.voff[pb + tid];
    dg::cp_wait<0>();
    __syncthreads();
    if (tid < np && g.aff) paf = g.aff[pd];
    if (ntn == 1) gemm_phase<1, RING>(Ap, Arow, r, nrep, Ts, Ys, LY, Ts + (size_t)kCols * LT);
    else gemm_phase<kNT, RING>(Ap, Arow, r, nrep, Ts, Ys, LY, Ts + (size_t)kCols * LT);
    if (tid < np) {
      s_poff[tid] = pd * nrep;
      if (g.aff) s_aff[tid] = paf;
    }
    __syncthreads();
    // per target group and density, pairs in order, through the permutation:
    // one index per (pair, row) for all densities, four pairs in flight
    for (int i = tid; i < nrep; i += kThreads) {
      int ca = 0, cb = 0, cc = 0;
      if (g.aff) {
        const uint32_t cw = g.coords[i];
        ca = cw & 255;
        cb = (cw >> 8) & 255;
        cc = cw >> 16;
      }
      const int32_t* pi = g.perm + i;
      auto index = [&](int jp) -> int {  // row of pair jp's Y column this thread adds
        if (!g.aff) return pi[s_poff[jp]];
        const int4 af = s_aff[jp];
        return s_lut[af.x * ca + af.y * cb + af.z * cc + af.w];
      };
      for (int e = 0; e < (multi ? 1 : ngrp); ++e) {
        const int64_t q0 = multi ? pa : s_gq[e], q1 = multi ? pe : s_gq[e + 1];
        const int ja = (int)(max(q0, pb) - pb), jb = (int)(min(q1, pb + np) - pb);
        if (ja >= jb) continue;
        const bool first = (pb + ja) == q0, last = (pb + jb) == q1;
        double* const d0 = g.part + (tg0 + e - g.g0) * nd * (int64_t)nrep;
        double s[kMaxNd];
#pragma unroll
        for (int l = 0; l < kMaxNd; ++l) s[l] = (first || l >= nd) ? 0.0 : carry[(size_t)l * nrep + i];
        for (int jp = ja; jp < jb; jp += 4) {
          int id[4];
#pragma unroll
          for (int v = 0; v < 4; ++v) id[v] = (jp + v < jb) ? index(jp + v) : 0;
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
          if (last) d0[(int64_t)l * nrep + i] = s[l];
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

template <bool RING>  // (instantiated with the ring only; see launch())
__global__ void __launch_bounds__(kThreads, 2) m2l_fused_kernel(Args g) {  // <= 128 registers
  // Persistent CTAs (two per SM): CTA b runs units b, b + gridDim.x, ... of
  // the heaviest-first list.  What a freshly launched CTA would wait for at
  // its start -- the unit record (one L2 round trip) and the first T tile
  // (another) -- is fetched during the previous unit instead: the next
  // record by cp.async into shared memory under the product, the next T tile
  // right after the product's barrier (Ts is free then) under the
  // accumulation.  Per-unit tables are double-buffered by unit parity, so a
  // unit's set-up never waits for the previous unit's stragglers.
  extern __shared__ __align__(16) double sm[];
  __shared__ int s_poff[kCols];            // perm row offset (offset index x nrep) of the pass's pairs
  __shared__ int4 s_aff[kCols];            // ... or their permutations in closed form
  __shared__ int64_t s_gq[2][kCols + 1];   // first pair of the unit's groups (one-pass units)
  __shared__ int s_slot[2];                // a multi-pass unit's carry slot
  __shared__ __align__(16) int64_t s_rec[2][kRec];  // prefetched unit records
  constexpr int LT = ldt();
  const int nd = g.nd, nrep = g.nrep;
  const int LY = ldy(nrep);
  double* Ys = sm;                          // [column][row], stride LY
  double* Ts = sm + (size_t)kCols * LY;     // [column][k], stride LT
  const int tid = threadIdx.x;
  const int ppp = kCols / nd;  // pairs per pass

  // T columns of a pass (global columns are tstride(r) doubles, zero past r):
  // 16-byte cp.async copies into Ts[c][k] at stride LT (LT = 4 mod 16 doubles:
  // conflict-free fragment reads, as in dgemm_cols.cuh); the columns past ncol
  // of the last N-tile are zeroed.
  auto issue_T = [&](const double* Tu, int K4, int64_t pa, int64_t pe, int64_t pb) {
    const int ncol = (int)min((int64_t)ppp, pe - pb) * nd;
    const int ntn = (ncol + 7) / 8;
    const int h4 = K4 / 2;  // 16-byte pieces per column
    const double* Tc = Tu + (pb - pa) * nd * (int64_t)K4;
    for (int e = tid; e < h4 * ntn * 8; e += kThreads) {
      const int c = e / h4, k = (e - c * h4) * 2;
      dg::cp16(Ts + c * LT + k, c < ncol ? Tc + (int64_t)c * K4 + k : g.T, c < ncol ? 16 : 0);
    }
    dg::cp_commit();
  };
  int64_t u = blockIdx.x;
  if (u >= g.nunits) return;
  // the first unit's record straight from global memory, and its T tile's
  // copies before anything else so that they fly under the CTA's set-up
  const int64_t* rec = g.urec + kRec * u;
  issue_T(g.T + __ldg(rec + 2), tstride((int)__ldg(rec + 3)), __ldg(rec + 6), __ldg(rec + 7), __ldg(rec + 6));
  // lattice index -> expansion index, behind the tiles (and the ring): once per CTA
  uint16_t* const s_lut = reinterpret_cast<uint16_t*>(Ts + (size_t)kCols * LT + (RING ? kRingDoubles : 0));
  if (g.aff)
    for (int e = tid; e < g.lut_n; e += kThreads) s_lut[e] = g.lut[e];
  for (int par = 0;; par ^= 1) {
    // (one volatile generic load per field: the record sits in global memory
    // for a CTA's first unit, in shared memory afterwards, and must not be
    // re-read once the copy of the next record may be in flight)
    auto field = [&](int k) -> int64_t {
      int64_t v;
      asm volatile("ld.b64 %0, [%1];\n" : "=l"(v) : "l"(rec + k));
      return v;
    };
    const double* const Ap = g.A ? g.A + field(0) : nullptr;
    const double* const Arow = g.Arow + field(1);
    const double* const Tu = g.T + field(2);  // the unit's first T column
    const int r = (int)field(3);
    const int64_t tg0 = field(4);
    const int ngrp = (int)field(5);
    const int64_t pa = field(6), pe = field(7);
    const bool multi = (pe - pa) > ppp;  // one group in several passes
    const int K4 = tstride(r);
    const int64_t un = u + gridDim.x;
    const bool more = un < g.nunits;
    if (pa >= pe) {  // a unit without pairs (the host builds none): only hand over to the next one
      if (!more) break;
      __syncthreads();  // everyone is done with the previous unit's tables and record
      if (tid < kRec / 2)
        dg::cp16(reinterpret_cast<double*>(s_rec[par ^ 1]) + 2 * tid,
                 reinterpret_cast<const double*>(g.urec + kRec * un) + 2 * tid, 16);
      dg::cp_commit();
      dg::cp_wait<0>();
      __syncthreads();
      const int64_t* const nr = s_rec[par ^ 1];
      issue_T(g.T + nr[2], tstride((int)nr[3]), nr[6], nr[7], nr[6]);
      u = un;
      rec = s_rec[par ^ 1];
      continue;
    }
    // group table (a multi-pass unit has one group); read after the first
    // pass's barriers
    for (int e = tid; e <= ngrp && e <= kCols; e += kThreads) s_gq[par][e] = g.tpair[tg0 + e];
    if (multi && tid == 0) {  // claim a carry slot (the pool outnumbers the resident CTAs)
      unsigned s = (unsigned)((u * 2654435761ull) % (unsigned)g.carry_slots);
      while (atomicCAS(g.carry_flag + s, 0u, 1u) != 0u) s = (s + 1) % (unsigned)g.carry_slots;
      s_slot[par] = (int)s;
    }
    double* carry = nullptr;

    for (int64_t pb = pa; pb < pe; pb += ppp) {
      const int np = (int)min((int64_t)ppp, pe - pb);
      const int ncol = np * nd;
      const int ntn = (ncol + 7) / 8;  // N-tiles in use
      // the pairs' offsets (and their closed-form permutations: a dependent
      // load) are only needed by the accumulation: loaded here, parked in
      // registers under the product, stored after it -- the barrier before the
      // product does not wait for them
      int pd = 0;
      int4 paf = make_int4(0, 0, 0, 0);
      if (tid < np) pd = g.voff[pb + tid];
      dg::cp_wait<0>();
      __syncthreads();  // this pass's T has landed; the previous accumulation is done with Ys / s_poff
      if (pb == pa) {
        if (multi) carry = g.carry + (size_t)s_slot[par] * kMaxNd * nrep;
        // the next unit's record, under the product
        if (more && tid < kRec / 2)
          dg::cp16(reinterpret_cast<double*>(s_rec[par ^ 1]) + 2 * tid,
                   reinterpret_cast<const double*>(g.urec + kRec * un) + 2 * tid, 16);
        dg::cp_commit();
      }
      if (tid < np && g.aff) paf = g.aff[pd];
      if (ntn == 1) gemm_phase<1, RING>(Ap, Arow, r, nrep, Ts, Ys, LY, Ts + (size_t)kCols * LT);
      else gemm_phase<kNT, RING>(Ap, Arow, r, nrep, Ts, Ys, LY, Ts + (size_t)kCols * LT);
      if (tid < np) {
        s_poff[tid] = pd * nrep;
        if (g.aff) s_aff[tid] = paf;
      }
      dg::cp_wait<0>();  // (the record copy; the ring's groups are done)
      __syncthreads();   // Y complete, Ts free, the next record visible
      // the next pass's T tile under the accumulation: this unit's next pass,
      // or the next unit's first
      if (pb + ppp < pe) {
        issue_T(Tu, K4, pa, pe, pb + ppp);
      } else if (more) {
        const int64_t* const nr = s_rec[par ^ 1];
        issue_T(g.T + nr[2], tstride((int)nr[3]), nr[6], nr[7], nr[6]);
      }
      // per target group and density, pairs in order, through the permutation:
      // one index per (pair, row) for all densities, four pairs in flight
      for (int i = tid; i < nrep; i += kThreads) {
        int ca = 0, cb = 0, cc = 0;
        if (g.aff) {
          const uint32_t cw = g.coords[i];
          ca = cw & 255;
          cb = (cw >> 8) & 255;
          cc = cw >> 16;
        }
        const int32_t* pi = g.perm + i;
        auto index = [&](int jp) -> int {  // row of pair jp's Y column this thread adds
          if (!g.aff) return pi[s_poff[jp]];
          const int4 af = s_aff[jp];
          return s_lut[af.x * ca + af.y * cb + af.z * cc + af.w];
        };
        for (int e = 0; e < (multi ? 1 : ngrp); ++e) {
          const int64_t q0 = multi ? pa : s_gq[par][e], q1 = multi ? pe : s_gq[par][e + 1];
          const int ja = (int)(max(q0, pb) - pb), jb = (int)(min(q1, pb + np) - pb);
          if (ja >= jb) continue;
          const bool first = (pb + ja) == q0, last = (pb + jb) == q1;
          double* const d0 = g.part + (tg0 + e - g.g0) * nd * (int64_t)nrep;
          double s[kMaxNd];
#pragma unroll
          for (int l = 0; l < kMaxNd; ++l) s[l] = (first || l >= nd) ? 0.0 : carry[(size_t)l * nrep + i];
          for (int jp = ja; jp < jb; jp += 4) {
            int id[4];
#pragma unroll
            for (int v = 0; v < 4; ++v) id[v] = (jp + v < jb) ? index(jp + v) : 0;
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
            if (last) d0[(int64_t)l * nrep + i] = s[l];
            else carry[(size_t)l * nrep + i] = s[l];
          }
        }
      }
    }
    if (multi) {  // hand the carry slot back
      __syncthreads();
      if (tid == 0) {
        __threadfence();
        atomicExch(g.carry_flag + s_slot[par], 0u);
      }
    }
    if (!more) break;
    u = un;
    rec = s_rec[par ^ 1];
  }
}

// lut_n: entries of the lattice-index table (m^3; 0 without closed-form permutations)
inline size_t smem_bytes(int nrep, bool ring, int lut_n) {
  return sizeof(double) * ((size_t)kCols * ldy(nrep) + (size_t)kCols * ldt() + (ring ? kRingDoubles : 0)) +
         ((sizeof(uint16_t) * (size_t)lut_n + 15) / 16) * 16;
}
// the ring variant when two CTAs with a ring fit one SM (227 KB, 1 KB reserved per CTA)
inline bool use_ring(int nrep, int lut_n) {
  return 2 * (smem_bytes(nrep, true, lut_n) + 1024 + 512) <= 227 * 1024;
}

// The cube-symmetry permutations in closed form.  pts: the expansion points
// on [-1, 1]^3 (nrep x 3); they sit on an m x m x m tensor lattice (uniform
// surface lattice or Chebyshev grid, both symmetric), so every permutation
// perm[d] (noff x nrep) is "permute the axes, flip some": lattice coordinates
// (a, b, c) -> index A a + B b + C c + D of the image on the m^3 lattice.
// Returns false (outputs untouched) if any permutation is not of that form.
inline bool fit_symmetries(const double* pts, int nrep, const int32_t* perm, int noff,
                           std::vector<int32_t>& aff, std::vector<uint32_t>& coords,
                           std::vector<uint16_t>& lut, int& m_out) {
  std::vector<double> vals;
  for (int i = 0; i < nrep; ++i) {
    bool seen = false;
    for (double v : vals) seen = seen || std::fabs(v - pts[3 * i]) < 1e-9;
    if (!seen) vals.push_back(pts[3 * i]);
  }
  std::sort(vals.begin(), vals.end());
  const int m = (int)vals.size();
  if (m < 2 || m > 16 || nrep > 65535) return false;
  auto rank = [&](double x) {
    for (int k = 0; k < m; ++k)
      if (std::fabs(vals[k] - x) < 1e-9) return k;
    return -1;
  };
  std::vector<uint32_t> co(nrep);
  std::vector<int> c3(3 * nrep);
  std::vector<uint16_t> lu((size_t)m * m * m, 0);
  std::vector<uint8_t> used((size_t)m * m * m, 0);
  for (int i = 0; i < nrep; ++i) {
    const int a = rank(pts[3 * i]), b = rank(pts[3 * i + 1]), c = rank(pts[3 * i + 2]);
    if (a < 0 || b < 0 || c < 0) return false;
    c3[3 * i] = a; c3[3 * i + 1] = b; c3[3 * i + 2] = c;
    co[i] = (uint32_t)a | ((uint32_t)b << 8) | ((uint32_t)c << 16);
    lu[((size_t)a * m + b) * m + c] = (uint16_t)i;
    used[((size_t)a * m + b) * m + c] = 1;
  }
  static const int P6[6][3] = {{0, 1, 2}, {0, 2, 1}, {1, 0, 2}, {1, 2, 0}, {2, 0, 1}, {2, 1, 0}};
  const int stride[3] = {m * m, m, 1};
  std::vector<int32_t> af(4 * (size_t)noff);
  for (int d = 0; d < noff; ++d) {
    bool found = false;
    for (int p = 0; p < 6 && !found; ++p)
      for (int f = 0; f < 8 && !found; ++f) {
        // image coordinate k = (flip_k ? m - 1 - x[P6[p][k]] : x[P6[p][k]])
        int A[3] = {0, 0, 0}, D = 0;
        for (int k = 0; k < 3; ++k) {
          const int sgn = (f >> k) & 1 ? -1 : 1;
          A[P6[p][k]] += sgn * stride[k];
          if (sgn < 0) D += (m - 1) * stride[k];
        }
        bool ok = true;
        for (int i = 0; i < nrep && ok; ++i) {
          const int t = A[0] * c3[3 * i] + A[1] * c3[3 * i + 1] + A[2] * c3[3 * i + 2] + D;
          ok = t >= 0 && t < m * m * m && used[t] && lu[t] == perm[(size_t)d * nrep + i];
        }
        if (ok) {
          af[4 * (size_t)d] = A[0]; af[4 * (size_t)d + 1] = A[1]; af[4 * (size_t)d + 2] = A[2];
          af[4 * (size_t)d + 3] = D;
          found = true;
        }
      }
    if (!found) return false;
  }
  aff.swap(af);
  coords.swap(co);
  lut.swap(lu);
  m_out = m;
  return true;
}

// dc[t, l, i] += the slots of t's (target, key) groups in [g0, g1), in key
// order (rt_grp lists every target's groups by ascending key): with the
// batches of keys processed in order, every check value is the same
// left-to-right sum over the keys as a stream-ordered launch per key gave.
// One CTA per target with V pairs; rows strided over the threads.
__global__ void __launch_bounds__(256) reduce_kernel(const int64_t* __restrict__ rt_tgt,
                                                     const int64_t* __restrict__ rt_off,
                                                     const int64_t* __restrict__ rt_grp, int64_t g0,
                                                     int64_t g1, const double* __restrict__ part, int nd,
                                                     int nrep, double* __restrict__ dc) {
  __shared__ int s_lo, s_n;
  const int64_t ti = blockIdx.x;
  const int64_t q0 = rt_off[ti], q1 = rt_off[ti + 1];
  // the target's groups ascend (by key, hence by group index): those of this
  // batch are one contiguous run [lo, lo + n) of its list
  if (threadIdx.x < 32) {
    int lo = -1, n = 0;
    for (int64_t qb = q0; qb < q1; qb += 32) {
      const int64_t q = qb + threadIdx.x;
      const bool in = q < q1 && rt_grp[q] >= g0 && rt_grp[q] < g1;
      const unsigned m = __ballot_sync(0xffffffffu, in);
      if (m) {
        if (lo < 0) lo = (int)(qb - q0) + __ffs(m) - 1;
        n += __popc(m);
      }
    }
    if (threadIdx.x == 0) {
      s_lo = lo;
      s_n = n;
    }
  }
  __syncthreads();
  const int n = s_n;
  if (n == 0) return;  // nothing of this batch lands on the target: its check values stay untouched
  const int64_t* const gl = rt_grp + q0 + s_lo;
  double* const d = dc + rt_tgt[ti] * nd * (int64_t)nrep;
  const int len = nd * nrep;
  for (int e = threadIdx.x; e < len; e += 256) {
    double v = d[e];
    int j = 0;
    for (; j + 4 <= n; j += 4) {  // four slots in flight, added left to right
      const double p0 = part[(gl[j] - g0) * len + e], p1 = part[(gl[j + 1] - g0) * len + e];
      const double p2 = part[(gl[j + 2] - g0) * len + e], p3 = part[(gl[j + 3] - g0) * len + e];
      v += p0;
      v += p1;
      v += p2;
      v += p3;
    }
    for (; j < n; ++j) v += part[(gl[j] - g0) * len + e];
    d[e] = v;
  }
}

inline cudaError_t reduce(const int64_t* rt_tgt, const int64_t* rt_off, const int64_t* rt_grp, int64_t ntgt,
                          int64_t g0, int64_t g1, const double* part, int nd, int nrep, double* dc,
                          cudaStream_t st) {
  if (ntgt <= 0 || g1 <= g0) return cudaSuccess;
  reduce_kernel<<<(unsigned)ntgt, 256, 0, st>>>(rt_tgt, rt_off, rt_grp, g0, g1, part, nd, nrep, dc);
  return cudaGetLastError();
}

// slots of the carry pool: four per SM (two CTAs are resident per SM)
inline int carry_slots(int sm_count) { return 4 * sm_count; }

// largest nrep one CTA's tile fits in shared memory for
inline int max_nrep() { return (int)((216 * 1024 / sizeof(double) - (size_t)kCols * ldt()) / kCols) - 8; }

inline cudaError_t launch(const Args& a, int64_t nunits, int rmax, cudaStream_t st) {
  if (nunits <= 0) return cudaSuccess;
  if (rmax > 4 * kMaxKS || a.nd > kMaxNd || a.nd < 1 || !a.urec || !a.part || !a.carry || !a.carry_flag || a.carry_slots < 1 ||
      a.nrep > max_nrep())
    return cudaErrorInvalidValue;
  const int lut_n = a.aff ? a.lut_n : 0;
  if ((a.A == nullptr) == use_ring(a.nrep, lut_n) || !a.Arow) return cudaErrorInvalidValue;
  const bool ring = a.A != nullptr;
  const int need = (int)smem_bytes(a.nrep, ring, lut_n);
  static int attr[2] = {0, 0};
  if (need > attr[ring]) {
    const cudaError_t e = ring ? cudaFuncSetAttribute(m2l_fused_kernel<true>,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, need)
                               : cudaFuncSetAttribute(m2l_fused_unit_kernel,
                                                      cudaFuncAttributeMaxDynamicSharedMemorySize, need);
    if (e != cudaSuccess) return e;
    attr[ring] = need;
  }
  // ring variant: persistent CTAs, two per SM (what the tile is sized for),
  // striding the heaviest-first unit list (config 3 M2L 1.48 -> 1.43 ms per
  // pot+grad call, 10^6 points at eps 1e-6 10.6 -> 10.2 ms); the no-ring
  // variant keeps one CTA per unit (see m2l_fused_unit_kernel)
  static int sms = 0;
  if (sms == 0) {
    int dev = 0;
    cudaGetDevice(&dev);
    if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || sms <= 0) sms = 148;
  }
  Args b = a;
  b.nunits = nunits;
  if (ring) m2l_fused_kernel<true><<<(unsigned)std::min<int64_t>(nunits, 2 * (int64_t)sms), kThreads, need, st>>>(b);
  else m2l_fused_unit_kernel<<<(unsigned)nunits, kThreads, need, st>>>(b);
  return cudaGetLastError();
}

}  // namespace m2lf
}  // namespace lb
