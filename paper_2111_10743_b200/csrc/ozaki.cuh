// Emulated-fp64 GEMM on the 5th-gen tensor cores (tcgen05.mma kind::i8).
//
// Y (nrep x ncol, col-major fp64) = A (nrep x nrep, fp64) * X (nrep x ncol)
// by the Ozaki splitting: every row of A and every column of X is scaled by a
// power of two and written as S signed 7-bit slices,
//     A[r,k] = rs[r] * sum_i a_i[r,k] 2^{-7i},   X[k,c] = cs[c] * sum_j b_j[k,c] 2^{-7j},
// |a_i|, |b_j| <= 64.  The products a_i b_j with i + j = d < S are exact in
// int32 (K * 64 * 64 * S < 2^31 for K <= 8192) and accumulate into one TMEM
// accumulator per diagonal d; the epilogue sums the S diagonals in fp64
// (Horner in 2^{-7}) and applies rs[r] cs[c].  The dropped terms i + j >= S
// bound the error by about S 2^{-7S} max|A[r,:]| max|X[:,c]| K, so S = 8
// reaches fp64 roundoff and smaller S trade accuracy for speed.
//
// Layout:
//   A pack: [m tile (128 rows)][k chunk (32)][slice][4096 B]
//   B pack: [n tile (NT cols)][k chunk (32)][slice][NT * 32 B]
// both K-major SWIZZLE_NONE canonical core matrices (8 rows x 16 B = 128
// contiguous bytes; the two 16-B K halves LBO = 128 B apart, 8-row groups
// SBO = 256 B apart), so one pipeline stage is two bulk copies.
//
// Kernel: one CTA per (m tile, n tile), 6 warps: warp 0 streams the stages
// into shared memory (cp.async.bulk completing on an mbarrier); warp 1
// allocates TMEM and one lane issues, per k chunk, S tcgen05.cp (A slices
// shared -> TMEM) and the S(S+1)/2 MMAs (128 x NT x 32, A from TMEM, B from
// shared memory); warps 2-5 drain the accumulators (tcgen05.ld 32x32b) into
// fp64.
#pragma once

#include <cuda_runtime.h>
#include <cmath>
#include <cstdint>
#include <type_traits>

namespace lb {
namespace oz {

constexpr int kBM = 128;             // rows per tile (MMA M)
constexpr int kBK = 32;              // K per MMA (kind::i8)
constexpr int kABytes = kBM * kBK;   // one slice of one A stage

// Tiling per slice count.  The accumulators of one pass (G diagonals of NT
// TMEM columns) plus two A stages of 8 S columns must fit the 512 TMEM
// columns; every tcgen05.mma carries a fixed issue cost (~25 cycles measured)
// on top of 0.5 cycle per N column, so wide N with several passes over K
// (each pass accumulates a range of diagonals, the epilogue warps carry the
// fp64 partial sums across passes in registers) beats one narrow pass.
// pass_end(S, p): first diagonal after pass p.
__host__ __device__ constexpr int nt_for(int S) { return S <= 6 ? 128 : 96; }
__host__ __device__ constexpr int npass_for(int S) { return S <= 3 ? 1 : 2; }
__host__ __device__ constexpr int pass_end(int S, int p) {
  return npass_for(S) == 1 || p > 0 ? S : (S == 4 ? 2 : S <= 6 ? 3 : 4);
}
__host__ __device__ constexpr int stage_bytes(int S, int NT) { return S * (kABytes + NT * kBK); }
__host__ __device__ constexpr int stages_for(int S, int NT) {
  return stage_bytes(S, NT) * 6 <= 200 * 1024 ? 6
         : stage_bytes(S, NT) * 5 <= 200 * 1024 ? 5
         : stage_bytes(S, NT) * 4 <= 200 * 1024 ? 4 : 3;
}
__host__ __device__ constexpr size_t smem_bytes(int S, int NT) { return (size_t)stages_for(S, NT) * stage_bytes(S, NT); }

// byte offset of element (row r within its 128/64 tile, k within its 32 chunk)
// inside one slice block of the canonical layout
__host__ __device__ inline int core_offset(int r, int k) {
  return (r >> 3) * 256 + ((k >> 4) & 1) * 128 + (r & 7) * 16 + (k & 15);
}

// power-of-two scale so |v| * 2^{6-e} <= 64: returns e (0 for an all-zero row)
__host__ __device__ inline int slice_exponent(double amax) {
  if (!(amax > 0.0)) return 0;
  int e;
  (void)frexp(amax, &e);  // amax = f 2^e, f in [0.5, 1)
  return e;
}

// host: A (nrep x nrep, row-major) -> A pack + row scales (Mpad rows)
template <int S>
void pack_rows_host(const double* A, int nrep, uint8_t* pack, double* rs) {
  const int KC = (nrep + kBK - 1) / kBK, MT = (nrep + kBM - 1) / kBM;
  for (size_t i = 0; i < (size_t)MT * KC * S * kABytes; ++i) pack[i] = 0;
  for (int r = 0; r < MT * kBM; ++r) {
    if (r >= nrep) { rs[r] = 0.0; continue; }
    double amax = 0.0;
    for (int k = 0; k < nrep; ++k) amax = fmax(amax, fabs(A[(size_t)r * nrep + k]));
    const int e = slice_exponent(amax);
    rs[r] = ldexp(1.0, e - 6);
    const int mt = r / kBM, rl = r % kBM;
    for (int k = 0; k < nrep; ++k) {
      double v = ldexp(A[(size_t)r * nrep + k], 6 - e);
      for (int s = 0; s < S; ++s) {
        const double a = nearbyint(v);
        pack[((size_t)(mt * KC + k / kBK) * S + s) * kABytes + core_offset(rl, k % kBK)] = (uint8_t)(int8_t)(int)a;
        v = (v - a) * 128.0;
      }
    }
  }
}

// device: npanel matrices A (npanel, nrep, nrep) row-major -> packs
// (npanel, MT, KC, S, 4096) + row scales (npanel, MT*128); one block per
// (padded row, panel).  Plan-time work.
__global__ void pack_rows_kernel(const double* __restrict__ A, int nrep, int S, uint8_t* __restrict__ pack,
                                 double* __restrict__ rs) {
  __shared__ double red[32];
  const int KC = (nrep + kBK - 1) / kBK, MT = (nrep + kBM - 1) / kBM;
  const int r = blockIdx.x, panel = blockIdx.y;
  const double* a = A + ((int64_t)panel * nrep + (r < nrep ? r : 0)) * nrep;
  double m = 0.0;
  if (r < nrep)
    for (int k = threadIdx.x; k < nrep; k += blockDim.x) m = fmax(m, fabs(a[k]));
  for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) m = fmax(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0) red[0] = m;
  }
  __syncthreads();
  const int e = slice_exponent(red[0]);
  if (threadIdx.x == 0) rs[(int64_t)panel * MT * kBM + r] = r < nrep ? ldexp(1.0, e - 6) : 0.0;
  const int mt = r / kBM, rl = r % kBM;
  uint8_t* base = pack + (int64_t)panel * MT * KC * S * kABytes;
  for (int k = threadIdx.x; k < KC * kBK; k += blockDim.x) {
    double v = (r < nrep && k < nrep) ? ldexp(a[k], 6 - e) : 0.0;
    for (int s = 0; s < S; ++s) {
      const double q = rint(v);
      base[((int64_t)(mt * KC + k / kBK) * S + s) * kABytes + core_offset(rl, k % kBK)] = (uint8_t)(int8_t)(int)q;
      v = (v - q) * 128.0;
    }
  }
}

inline size_t pack_rows_bytes(int nrep, int S) {
  const int KC = (nrep + kBK - 1) / kBK, MT = (nrep + kBM - 1) / kBM;
  return (size_t)MT * KC * S * kABytes;
}
inline size_t pack_cols_bytes(int nrep, int S, int64_t ncol, int NT) {
  const int KC = (nrep + kBK - 1) / kBK;
  return (size_t)((ncol + NT - 1) / NT) * KC * S * NT * kBK;
}
inline size_t pack_cols_bytes_max(int nrep, int64_t ncol) {
  size_t m = 0;
  for (int S = 3; S <= 8; ++S) {
    const size_t b = pack_cols_bytes(nrep, S, ncol, nt_for(S));
    m = b > m ? b : m;
  }
  return m;
}

// optional column gather of the M2L: column c = pair (p0 + c / nd), density l
// = c % nd; X[k, c] = up[(src * nd + l) * nrep + perm_inv[off * nrep + k]],
// column scale vscale[pair]
struct ColGather {
  const double* up;
  const int64_t* vsrc;
  const int32_t* voff;
  const double* vscale;
  const int32_t* perm_inv;
  int64_t p0;
  int nd;
};

// one block per 8 columns (one core-matrix group), 16 K per thread
template <int S, int NT>
__global__ void slice_cols_kernel(const double* __restrict__ X, int64_t ldx, int nrep, int64_t ncol,
                                  ColGather g, uint8_t* __restrict__ pack, double* __restrict__ cs) {
  __shared__ unsigned long long cmax[8];
  const int KC = (nrep + kBK - 1) / kBK;
  const int n8 = threadIdx.x & 7, kch = threadIdx.x >> 3;
  const int64_t col = (int64_t)blockIdx.x * 8 + n8;
  if (threadIdx.x < 8) cmax[threadIdx.x] = 0ull;
  __syncthreads();
  double v[16];
  const int k0 = kch * 16;
  double lmax = 0.0;
  double csc = 1.0;
  if (col < ncol) {
    const double* src;
    const int32_t* pv = nullptr;
    if (g.up) {
      const int64_t pi = g.p0 + col / g.nd;
      const int l = (int)(col % g.nd);
      src = g.up + (g.vsrc[pi] * g.nd + l) * (int64_t)nrep;
      pv = g.perm_inv + (int64_t)g.voff[pi] * nrep;
      csc = g.vscale[pi];
    } else {
      src = X + col * ldx;
    }
#pragma unroll
    for (int e = 0; e < 16; ++e) {
      const int k = k0 + e;
      v[e] = k < nrep ? src[pv ? pv[k] : k] : 0.0;
      lmax = fmax(lmax, fabs(v[e]));
    }
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e) v[e] = 0.0;
  }
  if (lmax > 0.0) atomicMax(&cmax[n8], (unsigned long long)__double_as_longlong(lmax));
  __syncthreads();
  const int ex = slice_exponent(__longlong_as_double((long long)cmax[n8]));
  if (kch == 0 && col < ncol) cs[col] = ldexp(1.0, ex - 6) * csc;
#pragma unroll
  for (int e = 0; e < 16; ++e) v[e] = ldexp(v[e], 6 - ex);
  const int64_t tile = col / NT;
  const int cl = (int)(col % NT);
  constexpr int kBBytes = NT * kBK;
  uint8_t* dst = pack + ((tile * KC + kch / 2) * S) * (int64_t)kBBytes + core_offset(cl, k0 % kBK);
#pragma unroll
  for (int s = 0; s < S; ++s) {
    uint32_t w[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t acc = 0;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const double a = rint(v[4 * q + b]);
        v[4 * q + b] = (v[4 * q + b] - a) * 128.0;
        acc |= ((uint32_t)(uint8_t)(int8_t)(int)a) << (8 * b);
      }
      w[q] = acc;
    }
    *reinterpret_cast<uint4*>(dst + (int64_t)s * kBBytes) = make_uint4(w[0], w[1], w[2], w[3]);
  }
}

// ---------------------------------------------------------------------------
// tcgen05 / mbarrier / bulk-copy primitives

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)), "r"(bytes) : "memory");
}
// bounded wait: a protocol bug traps instead of hanging the device
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  uint32_t done = 0;
  for (int it = 0; it < (1 << 24); ++it) {
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}\n"
        : "=r"(done)
        : "r"(su32(b)), "r"(parity)
        : "memory");
    if (done) return;
  }
  asm volatile("trap;");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          su32(dst)),
      "l"(src), "r"(bytes), "r"(su32(bar))
      : "memory");
}
__device__ __forceinline__ uint64_t smem_desc(const void* p) {
  // SWIZZLE_NONE K-major: LBO 128 B, SBO 256 B, version 1
  return (uint64_t)((su32(p) >> 4) & 0x3FFF) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | ((uint64_t)1 << 46);
}
// S32 accumulate, s8 x s8, both K-major, M = 128, N = NT
__host__ __device__ constexpr uint32_t idesc_i8(int NT) {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NT >> 3) << 17) | ((uint32_t)(kBM >> 4) << 24);
}

__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(bar))
               : "memory");
}

// COLL: 0 plain, 1 fill the A collector, 2 reuse it, 3 reuse it a last time
// (consecutive MMAs on the same A slice keep it in the tensor core's
// operand collector instead of re-reading TMEM)
template <int COLL>
__device__ __forceinline__ void mma_i8_ts(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc,
                                          uint32_t acc) {
#define LB_MMA_TS(Q)                                                                          \
  asm volatile("{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"                            \
               "tcgen05.mma.cta_group::1.kind::i8" Q " [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem_d), \
               "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc))
  if (COLL == 1) LB_MMA_TS(".collector::a::fill");
  else if (COLL == 2) LB_MMA_TS(".collector::a::use");
  else if (COLL == 3) LB_MMA_TS(".collector::a::lastuse");
  else LB_MMA_TS("");
#undef LB_MMA_TS
}
template <int D>
__host__ __device__ constexpr double ldexp_const() {  // 2^{-7 D}
  double r = 1.0;
  for (int i = 0; i < D; ++i) r *= 0.0078125;
  return r;
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}

__device__ __forceinline__ void cp_s2t_128x256b(uint32_t taddr, uint64_t sdesc) {
  asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// A operand from TMEM (lane = row, 4 int8 per 32-bit column): each k chunk's
// A slices are bulk-copied to shared memory with the B slices and moved to
// TMEM by tcgen05.cp, which the tensor pipe executes in order with the MMAs;
// consecutive MMAs on one A slice reuse it from the operand collector.
// Passes: pass p accumulates diagonals [pass_end(p-1), pass_end(p)) and needs
// the slice prefixes A_0.., B_0.. up to its last diagonal (one bulk copy
// each per chunk).  TMEM: G = max diagonals per pass accumulators of NT
// columns, then 2 A stages of S slices x 8 columns.
constexpr int kEpiWarps = 8;  // two per TMEM lane quadrant, each half of the columns
constexpr int kThreads = 64 + 32 * kEpiWarps;

__host__ __device__ constexpr int gmax_for(int S) {
  return npass_for(S) == 1 ? S : (pass_end(S, 0) > S - pass_end(S, 0) ? pass_end(S, 0) : S - pass_end(S, 0));
}

template <int S, int NT, int FAKE = 0>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_kernel(const uint8_t* __restrict__ Ap, const uint8_t* __restrict__ Bp, const double* __restrict__ rs,
                const double* __restrict__ cs, int nrep, int KC, int64_t ncol, int64_t ldy,
                double* __restrict__ Y) {
  constexpr int ST = stages_for(S, NT);
  constexpr int NP = npass_for(S);
  constexpr int G = gmax_for(S);
  constexpr int kBBytes = NT * kBK;
  constexpr int kA = S * kABytes, kB = S * kBBytes;  // full-prefix sizes in the packs
  constexpr int kStage = stage_bytes(S, NT);
  constexpr uint32_t kIdesc = idesc_i8(NT);
  constexpr uint32_t kAcol = G * NT;  // first A column
  static_assert(G * NT + 2 * S * 8 <= 512, "TMEM budget");
  static_assert(G <= 4, "int64 diagonal combine holds at most 4 diagonals");
  extern __shared__ __align__(128) uint8_t smem[];
  __shared__ __align__(8) uint64_t full[ST], empty[ST], accf, tfree;
  __shared__ uint32_t tmem_base;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // m tiles of one n tile are adjacent in launch order: the n tile's B pack is
  // read from HBM once, the (small) A pack stays in L2
  const int mt = blockIdx.x;
  const int64_t nt = blockIdx.y;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    mbar_init(&accf, 1);
    mbar_init(&tfree, 32 * kEpiWarps);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(su32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (warp == 0) {
    if (lane == 0) {
      const uint8_t* A = Ap + (int64_t)mt * KC * kA;
      const uint8_t* B = Bp + nt * KC * kB;
      int g = 0;
#pragma unroll 1
      for (int p = 0; p < NP; ++p) {
        const int d1 = p == 0 ? pass_end(S, 0) : pass_end(S, 1);
#pragma unroll 1
        for (int kc = 0; kc < KC; ++kc, ++g) {
          const int s = g % ST;
          if (g >= ST) mbar_wait(&empty[s], ((g / ST) - 1) & 1);
          uint8_t* sa = smem + (size_t)s * kStage;
          const uint32_t ab = d1 * kABytes, bb = d1 * kBBytes;
          mbar_expect_tx(&full[s], (FAKE == 1 ? 0 : ab) + (FAKE == 2 ? 0 : bb));
          if (FAKE != 1) bulk_g2s(sa, A + (int64_t)kc * kA, ab, &full[s]);
          if (FAKE != 2) bulk_g2s(sa + S * kABytes, B + (int64_t)kc * kB, bb, &full[s]);
        }
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    if (lane == 0) {
      int g = 0;
#pragma unroll 1
      for (int p = 0; p < NP; ++p) {
        if (p > 0) {  // the epilogue has drained the previous pass's accumulators
          mbar_wait(&tfree, (p - 1) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        }
#pragma unroll 1
        for (int kc = 0; kc < KC; ++kc, ++g) {
          const int s = g % ST;
          const uint32_t ta0 = tmem + kAcol + (uint32_t)((g & 1) * S * 8);
          mbar_wait(&full[s], (g / ST) & 1);
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const uint8_t* sa = smem + (size_t)s * kStage;
          const uint8_t* sb = sa + S * kABytes;
          if (FAKE != 4) {
            // the two passes are separate unrolled bodies: the (i, j) pair
            // lists are compile-time
            auto body = [&](auto P0, auto P1) {
              constexpr int d0 = decltype(P0)::value, d1 = decltype(P1)::value;
#pragma unroll
              for (int i = 0; i < d1; ++i) cp_s2t_128x256b(ta0 + (uint32_t)(i * 8), smem_desc(sa + i * kABytes));
#pragma unroll
              for (int i = 0; i < d1; ++i) {
                constexpr int dummy = 0;
                (void)dummy;
                const int jlo = d0 - i > 0 ? d0 - i : 0, jhi = d1 - i;  // j in [jlo, jhi)
                const uint32_t ta = ta0 + (uint32_t)(i * 8);
                const uint32_t acc = (kc > 0 || i > 0) ? 1u : 0u;
                const uint64_t db = smem_desc(sb);
                if (jhi - jlo == 1) {
                  mma_i8_ts<0>(tmem + (uint32_t)((i + jlo - d0) * NT), ta, db + (uint64_t)((jlo * kBBytes) >> 4),
                               kIdesc, acc);
                } else {
                  mma_i8_ts<1>(tmem + (uint32_t)((i + jlo - d0) * NT), ta, db + (uint64_t)((jlo * kBBytes) >> 4),
                               kIdesc, acc);
#pragma unroll
                  for (int j = jlo + 1; j < jhi - 1; ++j)
                    mma_i8_ts<2>(tmem + (uint32_t)((i + j - d0) * NT), ta, db + (uint64_t)((j * kBBytes) >> 4),
                                 kIdesc, acc);
                  mma_i8_ts<3>(tmem + (uint32_t)((i + jhi - 1 - d0) * NT), ta,
                               db + (uint64_t)(((jhi - 1) * kBBytes) >> 4), kIdesc, acc);
                }
              }
            };
            if constexpr (NP == 1) {
              body(std::integral_constant<int, 0>{}, std::integral_constant<int, S>{});
            } else {
              if (p == 0)
                body(std::integral_constant<int, 0>{}, std::integral_constant<int, pass_end(S, 0)>{});
              else
                body(std::integral_constant<int, pass_end(S, 0)>{}, std::integral_constant<int, pass_end(S, 1)>{});
            }
          }
          mma_commit(&empty[s]);
        }
        mma_commit(&accf);
      }
    }
    __syncwarp();
  } else {
    // epilogue: warp w drains TMEM lanes 32 (w % 4) .. +32 for column half
    // (w - 2) / 4; fp64 partial sums stay in registers across passes
    const int q = warp & 3;
    const int h = (warp - 2) >> 2;
    constexpr int kHalf = ((NT / 8 + 1) / 2) * 8;
    const int c0 = h * kHalf;
    const int nc = h ? NT - kHalf : kHalf;
    const uint32_t tl = tmem + ((uint32_t)(q * 32) << 16);
    double y[kHalf];
#pragma unroll
    for (int c = 0; c < kHalf; ++c) y[c] = 0.0;
#pragma unroll 1
    for (int p = 0; p < NP; ++p) {
      mbar_wait(&accf, p & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      auto drain = [&](auto P0, auto P1) {
        constexpr int d0 = decltype(P0)::value, d1 = decltype(P1)::value;
#pragma unroll
        for (int cg = 0; cg < kHalf; cg += 8) {
          if (FAKE == 3 || cg >= nc) break;
          uint32_t v[d1 - d0][8];
#pragma unroll
          for (int d = 0; d < d1 - d0; ++d)
            asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                         : "=r"(v[d][0]), "=r"(v[d][1]), "=r"(v[d][2]), "=r"(v[d][3]), "=r"(v[d][4]),
                           "=r"(v[d][5]), "=r"(v[d][6]), "=r"(v[d][7])
                         : "r"(tl + (uint32_t)(d * NT + c0 + cg)));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            // combine the pass's diagonals exactly in int64 (|acc| < 2^27, at
            // most 4 diagonals: |t| < 2^49), convert once by the 2^52 + 2^51
            // magic add (no I2F), weight 2^{-7 (d1 - 1)}
            long long t = (long long)(int32_t)v[0][j];
#pragma unroll
            for (int d = 1; d < d1 - d0; ++d) t = t * 128 + (long long)(int32_t)v[d][j];
            const double td = __longlong_as_double(t + 0x4338000000000000LL) - 6755399441055744.0;
            y[cg + j] = fma(td, ldexp_const<d1 - 1>(), y[cg + j]);
          }
        }
      };
      if constexpr (NP == 1) {
        drain(std::integral_constant<int, 0>{}, std::integral_constant<int, S>{});
      } else {
        if (p == 0)
          drain(std::integral_constant<int, 0>{}, std::integral_constant<int, pass_end(S, 0)>{});
        else
          drain(std::integral_constant<int, pass_end(S, 0)>{}, std::integral_constant<int, pass_end(S, 1)>{});
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      mbar_arrive(&tfree);
    }
    const int row = mt * kBM + q * 32 + lane;
    if (row < nrep && FAKE != 3) {
      const double rsc = rs[row];
#pragma unroll
      for (int c = 0; c < kHalf; ++c) {
        const int64_t col = nt * NT + c0 + c;
        if (c < nc && col < ncol) Y[col * ldy + row] = y[c] * rsc * cs[col];
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
  }
}

template <int S, int NT = nt_for(S)>
cudaError_t slice_cols(const double* X, int64_t ldx, int nrep, int64_t ncol, const ColGather* g,
                       uint8_t* pack, double* cs, cudaStream_t st) {
  if (ncol <= 0) return cudaSuccess;
  const int KC = (nrep + kBK - 1) / kBK;
  const int64_t ntile = (ncol + NT - 1) / NT;
  ColGather gg{};
  if (g) gg = *g;
  slice_cols_kernel<S, NT><<<(unsigned)(ntile * (NT / 8)), 16 * KC, 0, st>>>(X, ldx, nrep, ncol, gg, pack, cs);
  return cudaGetLastError();
}

template <int S, int NT = nt_for(S), int FAKE = 0>
cudaError_t gemm(const uint8_t* Ap, const uint8_t* Bp, const double* rs, const double* cs, int nrep,
                 int64_t ncol, double* Y, int64_t ldy, cudaStream_t st) {
  if (ncol <= 0) return cudaSuccess;
  // every CTA allocates all 512 TMEM columns: reserve enough shared memory
  // that a second CTA never lands on the SM (its tcgen05.alloc would stall)
  constexpr size_t kSmem = smem_bytes(S, NT) > 232448 / 2 + 1024 ? smem_bytes(S, NT) : 232448 / 2 + 1024;
  static bool attr = false;
  if (!attr) {
    const cudaError_t e =
        cudaFuncSetAttribute(gemm_kernel<S, NT, FAKE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)kSmem);
    if (e != cudaSuccess) return e;
    attr = true;
  }
  const int KC = (nrep + kBK - 1) / kBK, MT = (nrep + kBM - 1) / kBM;
  const int64_t ntile = (ncol + NT - 1) / NT;
  gemm_kernel<S, NT, FAKE><<<dim3((unsigned)MT, (unsigned)ntile), kThreads, kSmem, st>>>(Ap, Bp, rs, cs, nrep, KC, ncol,
                                                                              ldy, Y);
  return cudaGetLastError();
}

// runtime-S entry used by the FMM: slice (with the M2L gather) + GEMM
inline cudaError_t m2l_gemm(int S, const uint8_t* Ap, const double* rs, const ColGather& g, int nrep,
                            int64_t ncol, uint8_t* Bp, double* cs, double* Y, cudaStream_t st) {
  cudaError_t e = cudaErrorInvalidValue;
  switch (S) {
#define LB_OZ_CASE(SS)                                                        \
  case SS:                                                                    \
    e = slice_cols<SS>(nullptr, 0, nrep, ncol, &g, Bp, cs, st);               \
    if (e == cudaSuccess) e = gemm<SS>(Ap, Bp, rs, cs, nrep, ncol, Y, nrep, st); \
    break;
    LB_OZ_CASE(3)
    LB_OZ_CASE(4)
    LB_OZ_CASE(5)
    LB_OZ_CASE(6)
    LB_OZ_CASE(7)
    LB_OZ_CASE(8)
#undef LB_OZ_CASE
    default: break;
  }
  return e;
}

}  // namespace oz
}  // namespace lb
