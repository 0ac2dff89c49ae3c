// The GMRES operator apply on the device: LayerOperatorSet.apply_a1/a2/a3 and
// apply_layer (operators.py:126-266) as a fixed sequence of fused kernels:
//
//   oversample  : tau -> w_over * (over_interp @ tau_patch)  written straight
//                 into the packed far-field source records  (surface.py:370)
//   far         : one tiled fp64 all-pairs sweep per FMM call of the
//                 reference, computing ONLY the projections the operator
//                 consumes (pot, n.grad, n.H.n + n.grad_dipole, ...) rather
//                 than full grad/hess arrays (operators.py:237-259)
//   csr + epi   : the near-correction SpMVs of one pass share one read of the
//                 CSR pattern (all kinds share it, quadrature.py:693-700) and
//                 the scalar glue (1/4pi, -tau/4, 2H S', W-average) runs in
//                 the same kernel; the W-average is a deterministic grid
//                 reduction published on the device
//
// Signs/ordering follow the reference code (not the paper text) where they
// differ.
#include <algorithm>
#include <cmath>
#include <string>
#include <type_traits>
#include <vector>

#include "lb_common.cuh"
#include "opfar.cuh"
#include "reduce.cuh"

struct lb_fmm_plan;
namespace lb {  // fmm_plan.h (fmm_apply.cu): the two-density A3 call with a projected leaf stage
int fmm_apply_a3proj(lb_fmm_plan* P, const double* charges, const double* dipoles, const double* tnrm,
                     const double* snrm, double* pot, double* grad, double* hess, double* proj,
                     cudaStream_t st);
}

namespace lb {

// ---------------------------------------------------------------------------
// oversampling (interpolate_to_oversampled, surface.py:370-375) fused with the
// over_weights scaling and the write into the packed source records.  One
// block per patch.  Optionally adds a device scalar to input vector 0 in place
// first (A2's W-average, operators.py:212).

struct OvsArgs {
  const double* in[3];
  int slot[3];
  double scale[3];  // per-input factor folded into the record (FarA3c: 3 c1)
  int nv;
  double* in0_add_target;  // == in[0] when the scalar must be added, else null
  const double* add_scalar;
  double* pack;
  int S;
  const double* w_over;
  const double* oi;  // (nbo, nb)
  int nb, nbo;
};

__global__ void __launch_bounds__(128) oversample_kernel(OvsArgs a) {
  extern __shared__ double sv[];  // nv * nb
  const int64_t p = blockIdx.x;
  const int nb = a.nb;
  for (int k = threadIdx.x; k < a.nv * nb; k += blockDim.x) {
    const int v = k / nb, b = k - v * nb;
    double x = a.in[v][p * nb + b];
    if (v == 0 && a.in0_add_target) {
      x += a.add_scalar[0];
      a.in0_add_target[p * nb + b] = x;
    }
    sv[k] = x;
  }
  __syncthreads();
  for (int o = threadIdx.x; o < a.nbo; o += blockDim.x) {
    const double* row = a.oi + (int64_t)o * nb;
    const int64_t gi = p * a.nbo + o;
    const double w = a.w_over[gi];
    for (int v = 0; v < a.nv; ++v) {
      double s = 0.0;
      for (int b = 0; b < nb; ++b) s = fma(__ldg(row + b), sv[v * nb + b], s);
      a.pack[gi * a.S + a.slot[v]] = (w * a.scale[v]) * s;
    }
  }
}

// fill geometry slots of a packed record buffer ([x y z] or [x y z nx ny nz])
__global__ void fill_geom_kernel(const double* __restrict__ pos, const double* __restrict__ nrm,
                                 int64_t ns, int64_t ns_pad, int S, double* __restrict__ pack) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns_pad) return;
  double* r = pack + i * S;
  for (int k = 0; k < S; ++k) r[k] = 0.0;
  if (i >= ns) return;
  r[0] = pos[3 * i];
  r[1] = pos[3 * i + 1];
  r[2] = pos[3 * i + 2];
  if (nrm && S >= 8) {
    r[3] = nrm[3 * i];
    r[4] = nrm[3 * i + 1];
    r[5] = nrm[3 * i + 2];
  }
}

// ---------------------------------------------------------------------------
// CSR multi-job SpMV with a fused epilogue: one warp per row; every job reads
// the shared pattern once per nnz (repeated value/x reads of a pass hit L1).

template <int J>
struct CsrJobs {
  const double* val[J];  // the DISTINCT value arrays (Mix::K of them)
  const double* x[J];    // the DISTINCT densities (Mix::X of them)
};

// Job j of a pass multiplies value array vi(j) by density xi(j).  Distinct
// arrays are loaded once per nnz (A3's second pass reads S' for two densities
// and mu2 for three kinds: 3 value loads + 2 gathers instead of 4 + 4).
template <int J>
struct MixId {
  static constexpr int K = J, X = J;
  __host__ __device__ static constexpr int vi(int j) { return j; }
  __host__ __device__ static constexpr int xi(int j) { return j; }
};
template <int J>
struct MixOneX {  // J kinds applied to one density
  static constexpr int K = J, X = 1;
  __host__ __device__ static constexpr int vi(int j) { return j; }
  __host__ __device__ static constexpr int xi(int) { return 0; }
};
struct MixA3p2 {  // [S' mu1, S mu2, S' mu2, (S''+D') mu2]; vals {S', S, S''+D'}, xs {mu1, mu2}
  static constexpr int K = 3, X = 2;
  __host__ __device__ static constexpr int vi(int j) { return j == 0 ? 0 : (j == 1 ? 1 : (j == 2 ? 0 : 2)); }
  __host__ __device__ static constexpr int xi(int j) { return j == 0 ? 0 : 1; }
};
struct MixA3p2F {  // [S' mu1, S' mu2, (S''+D') mu2]; vals {S', S''+D'}, xs {mu1, mu2}
  static constexpr int K = 2, X = 2;
  __host__ __device__ static constexpr int vi(int j) { return j == 2 ? 1 : 0; }
  __host__ __device__ static constexpr int xi(int j) { return j == 0 ? 0 : 1; }
};

constexpr int kCsrBT = 256;
constexpr int kCsrRows = 8;  // rows per block: one warp per row (power of 2)

// Far-sweep partials (one per source split) are summed for the block's rows
// in a coalesced first phase (thread = row, fixed split order:
// deterministic) into shared memory; the epilogue reads them through f().
struct EpiBase {
  static constexpr int kMaxOut = 4;
  const double* part;
  SkLayout L;
  int nout;
  const double* fs;  // shared: fs[o * kCsrRows + local_row]
  int64_t row0;
  __device__ double f(int o, int64_t i) const { return fs[o * kCsrRows + (int)(i - row0)]; }
};

// generic: y_j = (accumulate ? y_j : 0) + acc_j
template <int J>
struct EpiStore {
  static constexpr bool kReduce = false;
  double* y[J];
  int accumulate;
  __device__ double operator()(int64_t i, const double* acc) const {
#pragma unroll
    for (int j = 0; j < J; ++j) y[j][i] = (accumulate ? y[j][i] : 0.0) + acc[j];
    return 0.0;
  }
};

// apply_layer: y = sign * far_o / 4pi + C tau  (operators.py:155)
struct EpiLayer : EpiBase {
  static constexpr bool kReduce = false;
  int o;
  double sign;
  double* y;
  __device__ double operator()(int64_t i, const double* acc) const {
    return (y[i] = fma(sign * kInv4Pi, f(o, i), acc[0])), 0.0;
  }
};

// A3 pass 1 (operators.py:239-241)
struct EpiA3p1 : EpiBase {
  static constexpr bool kReduce = false;
  double *s_tau, *sp_tau;
  __device__ double operator()(int64_t i, const double* acc) const {
    s_tau[i] = fma(f(0, i), kInv4Pi, acc[0]);
    sp_tau[i] = fma(-f(1, i), kInv4Pi, acc[1]);
    return 0.0;
  }
};

// A3 pass 1 with the W-average folded in: eta = <Phi, s_tau> / sum(w), where
// Phi = S^T w (lb_opset_set_eta_weights) so that <w, S mu2> = <Phi, mu2> and
// mu2 = s_tau is known here, one pass before the reference forms s_mu2
struct EpiA3p1R : EpiA3p1 {
  static constexpr bool kReduce = true;
  const double* phi;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double s = fma(f(0, i), kInv4Pi, acc[0]);
    s_tau[i] = s;
    sp_tau[i] = fma(-f(1, i), kInv4Pi, acc[1]);
    return phi[i] * s;
  }
};

// A3 pass 2 after the fused sweep (FarA3c): one far output, eta already
// reduced by pass 1 (scal[0]); corrections [S' mu1, S' mu2, (S''+D') mu2]
struct EpiA3p2F : EpiBase {
  static constexpr bool kReduce = false;
  const double *tau, *curv, *eta;
  double* result;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double corr = fma(-2.0 * curv[i], acc[1], acc[0] - acc[2]);
    result[i] = fma(-f(0, i), kInv4Pi, fma(tau[i], -0.25, corr)) + eta[0];
    return 0.0;
  }
};

// A3 pass 2 after the two-density FMM call (FK_A3M): far outputs
// [sp_mu1 - sppdp_mu2 - 2H sp_mu2 (x -4pi), S[mu2] far]; corrections as EpiA3p2
// (MixA3p2); reduces w * s_mu2 (eta is added by phase 2)
struct EpiA3p2M : EpiBase {
  static constexpr bool kReduce = true;
  const double *tau, *curv, *w;
  double* result;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double s_mu2 = fma(f(1, i), kInv4Pi, acc[1]);
    const double corr = fma(-2.0 * curv[i], acc[2], acc[0] - acc[3]);
    result[i] = fma(-f(0, i), kInv4Pi, fma(tau[i], -0.25, corr));
    return w[i] * s_mu2;
  }
};

// A3 pass 2 (operators.py:252-263) minus the eta term; reduces w * s_mu2
struct EpiA3p2 : EpiBase {
  static constexpr bool kReduce = true;
  const double *tau, *curv, *w;
  double* result;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double sp_mu1 = fma(-f(0, i), kInv4Pi, acc[0]);
    const double s_mu2 = fma(f(1, i), kInv4Pi, acc[1]);
    const double sp_mu2 = fma(-f(2, i), kInv4Pi, acc[2]);
    const double sppdp_mu2 = fma(f(3, i), kInv4Pi, acc[3]);
    result[i] = -tau[i] / 4.0 + sp_mu1 - sppdp_mu2 - 2.0 * curv[i] * sp_mu2;
    return w[i] * s_mu2;
  }
};

// A2 pass 1 (operators.py:204-212): mu1 = D tau, mu2 = -(S''+D')tau - 2H S'tau
// (+ ws added by the next oversample); reduces w * s_tau
struct EpiA2p1 : EpiBase {
  static constexpr bool kReduce = true;
  const double *curv, *w;
  double *mu1, *mu2;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double s_tau = fma(f(0, i), kInv4Pi, acc[0]);
    const double d_tau = fma(f(1, i), kInv4Pi, acc[1]);
    const double sp_tau = fma(-f(2, i), kInv4Pi, acc[2]);
    const double sppdp_tau = fma(f(3, i), kInv4Pi, acc[3]);
    mu1[i] = d_tau;
    mu2[i] = -sppdp_tau - 2.0 * curv[i] * sp_tau;
    return w[i] * s_tau;
  }
};

// A2 pass 2 (operators.py:222-224)
struct EpiA2p2 : EpiBase {
  static constexpr bool kReduce = false;
  const double* tau;
  double* result;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double d_mu1 = fma(f(0, i), kInv4Pi, acc[0]);
    const double s_mu2 = fma(f(1, i), kInv4Pi, acc[1]);
    result[i] = -tau[i] / 4.0 + s_mu2 + d_mu1;
    return 0.0;
  }
};

// A1 pass 1 (operators.py:169-179): s_tau for eta, grad S tau, tangential
// projection mu = g^{ij} x_i x_j . grad; reduces w * s_tau
struct EpiA1p1 : EpiBase {
  static constexpr bool kReduce = true;
  const double *tu, *tv, *gi, *w;
  double *mux, *muy, *muz;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double s_tau = fma(f(0, i), kInv4Pi, acc[0]);
    const double gx = fma(-f(1, i), kInv4Pi, acc[1]);
    const double gy = fma(-f(2, i), kInv4Pi, acc[2]);
    const double gz = fma(-f(3, i), kInv4Pi, acc[3]);
    const double* u = tu + 3 * i;
    const double* v = tv + 3 * i;
    const double* g = gi + 4 * i;
    const double gu = gx * u[0] + gy * u[1] + gz * u[2];
    const double gv = gx * v[0] + gy * v[1] + gz * v[2];
    const double a = g[0] * gu + g[1] * gv;
    const double b = g[2] * gu + g[3] * gv;
    mux[i] = a * u[0] + b * v[0];
    muy[i] = a * u[1] + b * v[1];
    muz[i] = a * u[2] + b * v[2];
    return w[i] * s_tau;
  }
};

// A1 pass 2 (operators.py:181-187): div + eta * phi0
struct EpiA1p2 : EpiBase {
  static constexpr bool kReduce = false;
  const double *phi0, *eta;
  double* result;
  __device__ double operator()(int64_t i, const double* acc) const {
    const double div_far = -f(0, i) * kInv4Pi;
    double div = 0.0;
    div += div_far + acc[0];
    div += acc[1];
    div += acc[2];
    result[i] = div + eta[0] * phi0[i];
    return 0.0;
  }
};

// One block = 8 warps = RB rows x W warps per row (W = wpr in {1,2,4,8},
// picked from the mean row length so every warp has ~4 chunks of 32 nnz in
// flight: the row loop is latency-bound otherwise).  Segment warps of a row
// combine their partial sums in a fixed order through shared memory.
// Three CTAs per SM by launch bounds (<= 85 registers).  Left to itself ptxas
// builds the row loop in 48 registers by interleaving the value loads with
// the FMAs that consume them, so an in-order warp has ~6 of its 16-24 loads
// in flight; with the larger budget it issues a whole unrolled iteration's
// loads first.  Config 3 (B200): pass 1 1.027 -> 0.947 ms, pass 2 1.439 ->
// 1.271 ms (5.5 / 6.1 TB/s of actual bytes; a pure two-stream read in the
// same row shape, lb_probe_read_rows, runs at 6.9).  Two CTAs per SM (96
// registers) lose it again (1.047 / 1.330), four (64) match three.
constexpr int kCsrMinBlocks = 3;
template <int J, class E, class Mix = MixId<J>>
__global__ void __launch_bounds__(kCsrBT, kCsrMinBlocks) csr_epi_kernel(const int64_t* __restrict__ indptr,
                                                         const int32_t* __restrict__ indices,
                                                         const int32_t* __restrict__ bstart, int bnb,
                                                         int64_t grow0, int64_t nrows, int wpr,
                                                         CsrJobs<J> jobs, E epi, double* partials,
                                                         unsigned* ticket, double* red_out,
                                                         double red_div) {
  // local rows r in [0, nrows) are global rows grow0 + r (sharded apply)
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  const int rb = (kCsrBT / 32) / wpr;
  const int64_t row0 = (int64_t)blockIdx.x * rb;
  __shared__ double fs[EpiBase::kMaxOut * kCsrRows];
  __shared__ double wacc[kCsrBT / 32][J];
  E e = epi;
  if constexpr (std::is_base_of<EpiBase, E>::value) {
    // all 256 threads: (row lr, output o) x 8 slot-lanes sl, then a fixed-order
    // 8-way reduction through shared memory (latency-bound otherwise)
    __shared__ double red8[8][EpiBase::kMaxOut * kCsrRows];
    const int lr = threadIdx.x & (kCsrRows - 1);
    const int o = (threadIdx.x >> 3) & 3;
    const int sl = threadIdx.x >> 5;
    double v = 0.0;
    const int64_t i = row0 + lr;
    if (lr < rb && o < e.nout && i < nrows) {
      const int64_t t = i / e.L.tt;
      const int lt = (int)(i - t * e.L.tt);
      const int64_t nseg = e.L.blast(t) - e.L.bfirst(t) + 1;
      for (int64_t k = sl; k < nseg; k += 8) v += e.part[e.L.idx(t, k, o, e.nout, lt)];
    }
    red8[sl][o * kCsrRows + lr] = v;
    __syncthreads();
    if (threadIdx.x < EpiBase::kMaxOut * kCsrRows) {
      double s8 = 0.0;
#pragma unroll
      for (int q = 0; q < 8; ++q) s8 += red8[q][threadIdx.x];
      fs[threadIdx.x] = s8;
    }
    e.fs = fs;
    e.row0 = grow0 + row0;
  }
  const int rloc = warp / wpr, seg = warp - rloc * wpr;
  const int64_t lrow = row0 + rloc;
  const int64_t row = grow0 + lrow;
  double acc[J];
#pragma unroll
  for (int j = 0; j < J; ++j) acc[j] = 0.0;
  if (lrow < nrows) {
    const int64_t kb = indptr[row], ke = indptr[row + 1];
    const int64_t stride = 32 * wpr;
    int64_t k = kb + seg * 32 + lane;
    constexpr int K = Mix::K, X = Mix::X;
    // column of entry k: the block-CSR index (one int32 start per block of
    // nb consecutive columns, quadrature.py:693-700: 4/nb bytes per entry)
    // when the handle has one, else the scalar index (4 bytes per entry).
    // A row is whole blocks, so entry k sits in block kb / nb + (k - kb) / nb:
    // one 64-bit division per row, then a 32-bit multiply-high per entry
    // (exact for k - kb < 2^32 / nb; rows hold at most cap * nb entries)
    const int64_t bbase = bstart ? kb / bnb : 0;
    const unsigned magic = bstart ? (unsigned)((0x100000000ull + bnb - 1) / (unsigned)bnb) : 0u;
    auto col = [&](int64_t kk) -> int {
      if (!bstart) return __ldg(indices + kk);
      const unsigned rel = (unsigned)(kk - kb);
      const unsigned q = __umulhi(rel, magic);
      return __ldg(bstart + bbase + q) + (int)(rel - q * (unsigned)bnb);
    };
    // loads in flight per lane: the value streams are the kernel's HBM
    // traffic, and fewer streams unroll deeper.  B200, config 3, with the
    // launch bounds above: two streams 6 / 8 / 10 / 12 / 16 entries -> 1.10 /
    // 0.947 / 0.981 / 1.07 / 1.35 ms; three streams 2 / 3 / 4 / 5 / 6 / 8 ->
    // 1.32 / 1.33 / 1.27 / 1.55 / 1.31 / 1.38 ms
    constexpr int UR = K >= 3 ? 4 : 8;
    for (; k + (UR - 1) * stride < ke; k += UR * stride) {
      int c[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) c[u] = col(k + stride * u);
      if constexpr (K >= 3) {  // three streams: per-entry loads
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          double v[K], xv[X];
#pragma unroll
          for (int q = 0; q < K; ++q) v[q] = __ldg(jobs.val[q] + k + stride * u);
#pragma unroll
          for (int q = 0; q < X; ++q) xv[q] = __ldg(jobs.x[q] + c[u]);
#pragma unroll
          for (int j = 0; j < J; ++j) acc[j] = fma(v[Mix::vi(j)], xv[Mix::xi(j)], acc[j]);
        }
      } else {
        double v[UR][K];
#pragma unroll
        for (int u = 0; u < UR; ++u)
#pragma unroll
          for (int q = 0; q < K; ++q) v[u][q] = __ldg(jobs.val[q] + k + stride * u);
#pragma unroll
        for (int u = 0; u < UR; ++u) {
          double xv[X];
#pragma unroll
          for (int q = 0; q < X; ++q) xv[q] = __ldg(jobs.x[q] + c[u]);
#pragma unroll
          for (int j = 0; j < J; ++j) acc[j] = fma(v[u][Mix::vi(j)], xv[Mix::xi(j)], acc[j]);
        }
      }
    }
    for (; k < ke; k += stride) {
      const int c = col(k);
      double v[K], xv[X];
#pragma unroll
      for (int q = 0; q < K; ++q) v[q] = __ldg(jobs.val[q] + k);
#pragma unroll
      for (int q = 0; q < X; ++q) xv[q] = __ldg(jobs.x[q] + c);
#pragma unroll
      for (int j = 0; j < J; ++j) acc[j] = fma(v[Mix::vi(j)], xv[Mix::xi(j)], acc[j]);
    }
#pragma unroll
    for (int j = 0; j < J; ++j) {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) acc[j] += __shfl_xor_sync(0xffffffffu, acc[j], o);
    }
    if (lane == 0) {
#pragma unroll
      for (int j = 0; j < J; ++j) wacc[warp][j] = acc[j];
    }
  }
  __syncthreads();
  double red = 0.0;
  if (lrow < nrows && seg == 0 && lane == 0) {
#pragma unroll
    for (int j = 0; j < J; ++j) {
      double t = 0.0;
      for (int q = 0; q < wpr; ++q) t += wacc[warp + q][j];
      acc[j] = t;
    }
    red = e(row, acc);
  }
  if constexpr (E::kReduce) grid_reduce_finish<kCsrBT>(red, partials, ticket, red_out, 0, red_div);
}

// warps per row from the mean row length.  Measured on B200 at config 2
// (617 nnz/row): 1 warp/row 33.6 us vs 4 warps/row 50 us for pass 1, so rows
// are only split when they are very long.
inline int csr_wpr(int64_t nnz, int64_t nrows) {
  const int64_t avg = nrows > 0 ? nnz / nrows : 0;
  return avg >= 8192 ? 4 : avg >= 4096 ? 2 : 1;
}

__global__ void add_scalar_kernel(double* y, int64_t n, const double* s) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] += s[0];
}

}  // namespace lb

// ===========================================================================
// the operator-set handle

struct lb_opset {
  lb_opset_desc d;
  int64_t r0 = 0, nr = 0;  // owned target rows [r0, r0 + nr) (sharded apply)
  double wsum = 0.0;
  int64_t ns_pad = 0;
  double* pack4 = nullptr;  // [x y z c]
  double* pack6 = nullptr;  // [x y z c0 c1 c2]
  double* pack8 = nullptr;  // [x y z nx ny nz c0 c1]
  double* part = nullptr;
  int64_t part_cap = 0;
  double* vec = nullptr;  // 8 work vectors of length n
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  double* scal = nullptr;  // [0] W-average / eta
  const double* phi_eta = nullptr;  // Phi = S^T w (global rows): fused A3 pass 2
  bool fmm_a3_two = true;  // FMM path: A3's second call on 2 densities (lb_opset_set_fmm_a3)
  int csr_blocks = 0;
  int csr_wpr = 1;
  int32_t* bstart = nullptr;  // block-CSR index: first column of every nb-block (nullptr: scalar)
  int bnb = 0;
  // optional FMM far field (lb_opset_set_fmm) and its scratch
  lb_fmm_plan* fmm = nullptr;
  bool timing = false;
  cudaEvent_t ev[16] = {};
  int nev = 0;
  double stage_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  double *f_ch = nullptr, *f_ch3 = nullptr, *f_dp = nullptr;
  double *f_pot = nullptr, *f_grad = nullptr, *f_hess = nullptr;
  double* f_proj = nullptr;  // (3, nt): projected leaf outputs of the 2-density A3 call
  int64_t fmm_nt = 0;        // the plan's targets: nr, or all n (replicated plan, owned range)
};

namespace lb {
namespace {

// launch shape per functor, from tools/far_sweep.cu on B200 (config-2 and
// 1e5-sized sweeps): 64-thread CTAs, 4 targets/thread with 64-source tiles for
// the light 4-double records, 2 targets/thread with 128-source tiles for the
// 8-double records; next source tile prefetched into registers.
constexpr int kFarBT = 64;

template <class F>
constexpr int far_tpt() {
  // FarA3a: 2 targets/thread with an 8-deep pair unroll (135 registers, 6
  // CTAs/SM): 381 vs 394 us at config 2 (tools/far_sweep.cu a3a, B200)
  return std::is_same<F, FarA3a>::value ? 2 : (F::S <= 4 && F::NOUT <= 2 ? 4 : 2);
}
template <class F>
constexpr int far_ur() {
  return std::is_same<F, FarA3a>::value || std::is_same<F, FarA3c>::value ? 8 : 4;
}
template <class F>
constexpr int far_ts() {
  // FarA3c: 64-source tiles with the 8-deep unroll, 654 vs 657.5 us (two runs)
  return F::S <= 4 || std::is_same<F, FarA3c>::value ? 64 : 128;
}
constexpr int kFarPad = 128;  // source padding: a multiple of every far_ts

template <class F>
SkLayout far_layout(const lb_opset* h) {
  constexpr int TPT = far_tpt<F>();
  static int per_sm = -1;
  if (per_sm < 0) {
    int b = 1;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, opfar_kernel<F, TPT, kFarBT, far_ts<F>(), true, far_ur<F>()>,
                                                  kFarBT, 0);
    per_sm = std::max(b, 1);
  }
  return make_sk_layout(h->nr, h->ns_pad, kFarBT * TPT, far_ts<F>(), (int64_t)sm_count() * per_sm);
}

template <class F>
int64_t far_part_size(const lb_opset* h) {
  const SkLayout L = far_layout<F>(h);
  return L.tiles * L.kmax * F::NOUT * L.tt;
}

template <class F>
int run_far(const lb_opset* h, const double* pack, SkLayout* out, cudaStream_t st) {
  constexpr int TPT = far_tpt<F>();
  const SkLayout L = far_layout<F>(h);
  if (L.tiles * L.kmax * F::NOUT * L.tt > h->part_cap)
    return fail(LB_ERR_ARG, "opset: partial buffer too small");
  opfar_kernel<F, TPT, kFarBT, far_ts<F>(), true, far_ur<F>()><<<(unsigned)L.G, kFarBT, 0, st>>>(
      h->d.nodes + 3 * h->r0, h->d.normals + 3 * h->r0, h->nr, pack, L, h->part,
      h->d.curvature ? h->d.curvature + h->r0 : nullptr);
  LB_CHECK_LAUNCH();
  *out = L;
  return LB_OK;
}

int oversample(const lb_opset* h, int nv, const double* const* in, const int* slot, double* pack,
               int S, bool add_ws, cudaStream_t st, const double* scale = nullptr) {
  OvsArgs a{};
  for (int v = 0; v < nv; ++v) {
    a.in[v] = in[v];
    a.slot[v] = slot[v];
    a.scale[v] = scale ? scale[v] : 1.0;
  }
  a.nv = nv;
  a.in0_add_target = add_ws ? const_cast<double*>(in[0]) : nullptr;
  a.add_scalar = h->scal;
  a.pack = pack;
  a.S = S;
  a.w_over = h->d.over_weights;
  a.oi = h->d.over_interp;
  a.nb = h->d.nb;
  a.nbo = h->d.nbo;
  oversample_kernel<<<(unsigned)h->d.npatches, 128, sizeof(double) * nv * h->d.nb, st>>>(a);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// vals: the pass's per-job value arrays, xs: per-job densities (J each);
// Mix collapses them to the distinct ones (the caller's order must match Mix)
template <int J, class E, class Mix = MixId<J>>
int run_csr(const lb_opset* h, const double* const* vals, const double* const* xs, const E& epi,
            cudaStream_t st, double red_div = 1.0) {
  CsrJobs<J> jobs{};
  for (int j = 0; j < J; ++j) {
    if (!vals[j]) return fail(LB_ERR_KEY, "opset: a required correction kind was not provided");
    jobs.val[Mix::vi(j)] = vals[j];
    jobs.x[Mix::xi(j)] = xs[j];
  }
  csr_epi_kernel<J, E, Mix><<<(unsigned)h->csr_blocks, kCsrBT, 0, st>>>(
      h->d.indptr, h->d.indices, h->bstart, h->bnb, h->r0, h->nr, h->csr_wpr, jobs, epi, h->partials, h->ticket,
      h->scal, red_div);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

template <class E>
E base_epi(const lb_opset* h, const SkLayout& L, int nout) {
  E e{};
  e.part = h->part;
  e.L = L;
  e.nout = nout;
  return e;
}

double* V(const lb_opset* h, int k) { return h->vec + (int64_t)k * h->d.n; }

// ---------------------------------------------------------------------------
// one far-field call of the reference (a `_far` call, operators.py:103-114):
// oversample the input vector(s) and run the sweep, either exact all-pairs
// (opfar_kernel) or through the attached FMM plan (lb_fmm_apply + a
// projection to the same per-target outputs), returning the partial layout
// the CSR epilogue reads.

enum FarKind { FK_S, FK_A3A, FK_A3B, FK_A2A, FK_A2B, FK_A1A, FK_A1B, FK_D, FK_A3C, FK_A3M };

struct FarSpec {
  double* pack;
  int S;
  int slot[3];
  double scale[3] = {1.0, 1.0, 1.0};
};

FarSpec far_spec(lb_opset* h, FarKind k) {
  switch (k) {
    case FK_S: case FK_A3A: case FK_A1A: return {h->pack4, 4, {3, 0, 0}};
    case FK_A3B: return {h->pack8, 8, {6, 7, 0}};
    case FK_A3C: return {h->pack8, 8, {6, 7, 0}, {1.0, 3.0, 1.0}};
    case FK_A2A: case FK_D: return {h->pack8, 8, {6, 0, 0}};
    case FK_A2B: return {h->pack8, 8, {7, 6, 0}};
    default: return {h->pack6, 6, {3, 4, 5}};  // FK_A1B
  }
}

int far_nout(FarKind k) {
  switch (k) {
    case FK_S: case FK_A1B: case FK_D: case FK_A3C: return 1;
    case FK_A3A: case FK_A2B: return 2;
    case FK_A3M: return 2;
    default: return 4;
  }
}

// sign * c * n_over dipoles for FMM densities
__global__ void dipole_kernel(const double* __restrict__ c, const double* __restrict__ nrm, int64_t ns,
                              double* __restrict__ out, double sign = 1.0) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ns) return;
  const double ci = sign * c[i];
  for (int k = 0; k < 3; ++k) out[3 * i + k] = ci * nrm[3 * i + k];
}

// FMM outputs -> the functor outputs, written as a one-segment stream-K layout
// pot/grad/hess/proj point at this handle's first row inside the plan's target
// arrays, whose per-density stride is ntp (= n for a plan on the handle's rows,
// = all nodes for a replicated plan with an owned-target range)
__global__ void project_kernel(int kind, const double* __restrict__ nrm, int64_t n, int64_t ntp,
                               const double* __restrict__ pot, const double* __restrict__ grad,
                               const double* __restrict__ hess, SkLayout L, int nout,
                               double* __restrict__ part, const double* __restrict__ curv,
                               const double* __restrict__ proj) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double nx = nrm[3 * i], ny = nrm[3 * i + 1], nz = nrm[3 * i + 2];
  auto ng = [&](int l) {  // n . grad_l
    const double* g = grad + ((int64_t)l * ntp + i) * 3;
    return nx * g[0] + ny * g[1] + nz * g[2];
  };
  auto nhn = [&](int l) {  // n . hess_l . n
    const double* H = hess + ((int64_t)l * ntp + i) * 9;
    return nx * (H[0] * nx + H[1] * ny + H[2] * nz) + ny * (H[3] * nx + H[4] * ny + H[5] * nz) +
           nz * (H[6] * nx + H[7] * ny + H[8] * nz);
  };
  double a[4] = {0, 0, 0, 0};
  switch (kind) {
    case FK_S: case FK_D: a[0] = pot[i]; break;
    case FK_A3A: a[0] = pot[i]; a[1] = -ng(0); break;
    case FK_A3B: a[0] = -ng(0); a[1] = pot[ntp + i]; a[2] = -ng(1); a[3] = nhn(1) + ng(2); break;
    // fused A3 call 2 on two FMM densities: X = (charge c0, dipole -c1 n) and
    // B = (charge c1): a0 = FarA3b's a0 + a3 - 2H a2 = -n.grad X + n.H_B.n + 2H n.grad B
    case FK_A3M: {  // + the projected leaf stage [-n.grad X + n.H_B.n, pot B, n.grad B]
      a[0] = fma(2.0 * curv[i], ng(1) + proj[2 * ntp + i], (nhn(1) - ng(0)) + proj[i]);
      a[1] = pot[ntp + i] + proj[ntp + i];
      break;
    }
    case FK_A2A: a[0] = pot[i]; a[1] = pot[ntp + i]; a[2] = -ng(0); a[3] = nhn(0) + ng(1); break;
    case FK_A2B: a[0] = pot[i]; a[1] = pot[ntp + i]; break;
    case FK_A1A:
      a[0] = pot[i];
      for (int k = 0; k < 3; ++k) a[1 + k] = -grad[i * 3 + k];
      break;
    case FK_A1B:
      a[0] = -(grad[(0 * ntp + i) * 3 + 0] + grad[(1 * ntp + i) * 3 + 1] + grad[(2 * ntp + i) * 3 + 2]);
      break;
  }
  const int64_t t = i / L.tt;
  const int lt = (int)(i - t * L.tt);
  for (int o = 0; o < nout; ++o) part[L.idx(t, 0, o, nout, lt)] = a[o];
}

int far_stage(lb_opset* h, FarKind kind, int nv, const double* const* in, bool add_ws, SkLayout* L,
              cudaStream_t st) {
  if (!h->fmm) {
    const FarSpec sp = far_spec(h, kind);
    LB_TRY(oversample(h, nv, in, sp.slot, sp.pack, sp.S, add_ws, st, sp.scale));
    switch (kind) {
      case FK_S: return run_far<FarS>(h, sp.pack, L, st);
      case FK_A3A: return run_far<FarA3a>(h, sp.pack, L, st);
      case FK_A3B: return run_far<FarA3b>(h, sp.pack, L, st);
      case FK_A3C: return run_far<FarA3c>(h, sp.pack, L, st);
      case FK_A2A: return run_far<FarA2a>(h, sp.pack, L, st);
      case FK_A2B: return run_far<FarA2b>(h, sp.pack, L, st);
      case FK_A1A: return run_far<FarA1a>(h, sp.pack, L, st);
      case FK_A1B: return run_far<FarA1b>(h, sp.pack, L, st);
      default: return run_far<FarD>(h, sp.pack, L, st);
    }
  }
  // FMM path: plain charge arrays c_v = w_over * oversample(in_v)
  const int64_t no = h->d.n_over, n = h->nr;
  const int slot[3] = {0, (int)no, (int)(2 * no)};
  LB_TRY(oversample(h, nv, in, slot, h->f_ch, 1, add_ws, st));
  double* c0 = h->f_ch;
  double* c1 = h->f_ch + no;
  double* ch = h->f_ch3;  // (3, no) densities handed to the FMM
  double* dp = h->f_dp;   // (3, no, 3)
  const unsigned g = (unsigned)ceil_div(no, 256);
  int nd = 1, level = 0;
  uint32_t cm = 0, dm = 0;
  const double* chp = c0;
  const double* dpp = nullptr;
  switch (kind) {
    case FK_S: nd = 1; cm = 1; level = 0; break;
    case FK_D:
      dipole_kernel<<<g, 256, 0, st>>>(c0, h->d.over_normals, no, dp);
      nd = 1; dm = 1; level = 0; chp = nullptr; dpp = dp; break;
    case FK_A3A: case FK_A1A: nd = 1; cm = 1; level = 1; break;
    case FK_A3B:  // charges [c0, c1, 0], dipoles [0, 0, c1 n]
      LB_CUDA(cudaMemcpyAsync(ch, c0, sizeof(double) * no, cudaMemcpyDeviceToDevice, st));
      LB_CUDA(cudaMemcpyAsync(ch + no, c1, sizeof(double) * no, cudaMemcpyDeviceToDevice, st));
      dipole_kernel<<<g, 256, 0, st>>>(c1, h->d.over_normals, no, dp + 2 * no * 3);
      nd = 3; cm = 3; dm = 4; level = 2; chp = ch; dpp = dp; break;
    case FK_A3M:  // charges [c0, c1] (f_ch already holds them), dipoles [-c1 n, 0]
      dipole_kernel<<<g, 256, 0, st>>>(c1, h->d.over_normals, no, dp, -1.0);
      nd = 2; cm = 3; dm = 1; level = 2; chp = c0; dpp = dp; break;
    case FK_A2A:  // charge c0 on density 0, dipole c0 n on density 1
      dipole_kernel<<<g, 256, 0, st>>>(c0, h->d.over_normals, no, dp + no * 3);
      nd = 2; cm = 1; dm = 2; level = 2; chp = c0; dpp = dp; break;
    case FK_A2B:  // dipole (w mu1) n on density 0, charge (w mu2) on density 1
      // in = {mu2, mu1}: c0 = w mu2, c1 = w mu1
      dipole_kernel<<<g, 256, 0, st>>>(c1, h->d.over_normals, no, dp);
      LB_CUDA(cudaMemcpyAsync(ch + no, c0, sizeof(double) * no, cudaMemcpyDeviceToDevice, st));
      nd = 2; cm = 2; dm = 1; level = 0; chp = ch; dpp = dp; break;
    case FK_A1B: nd = 3; cm = 7; level = 1; chp = c0; break;
  }
  LB_CHECK_LAUNCH();
  if (kind == FK_A3M) {  // projected leaf stage (fmm_plan.h: fmm_apply_a3proj)
    if (!h->f_proj) LB_CUDA(cudaMalloc((void**)&h->f_proj, sizeof(double) * 3 * std::max<int64_t>(h->fmm_nt, 1)));
    const double* tn = h->fmm_nt == h->nr ? h->d.normals + 3 * h->r0 : h->d.normals;
    const int rc = fmm_apply_a3proj(h->fmm, chp, dpp, tn, h->d.over_normals, h->f_pot, h->f_grad,
                                    h->f_hess, h->f_proj, st);
    if (rc != LB_OK) return fail(rc, std::string("far_stage(A3 two densities): ") + lb_last_error_string());
  } else {
    int rc = lb_fmm_apply(h->fmm, chp, dpp, nd, cm, dm, level, h->f_pot, h->f_grad, h->f_hess, st);
    if (rc != LB_OK) return fail(rc, std::string("far_stage(kind ") + std::to_string((int)kind) +
                                         "): " + lb_last_error_string());
  }
  SkLayout l1{};
  l1.tt = 64;
  l1.tiles = ceil_div(n, l1.tt);
  l1.C = 1;
  l1.U = l1.tiles;
  l1.G = l1.tiles;
  l1.kmax = 1;
  const int nout = far_nout(kind);
  const int64_t ntp = h->fmm_nt, toff = ntp == h->nr ? 0 : h->r0;
  project_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(
      (int)kind, h->d.normals + 3 * h->r0, n, ntp, h->f_pot + toff, h->f_grad + 3 * toff,
      h->f_hess + 9 * toff, l1, nout, h->part, h->d.curvature + h->r0, h->f_proj ? h->f_proj + toff : nullptr);
  LB_CHECK_LAUNCH();
  *L = l1;
  return LB_OK;
}

// The three formulations as phases separated by the only cross-row
// dependencies of the apply: a phase ends where every row's
// value of an intermediate density (or the W-average) is needed.  A sharded
// apply runs the phases on its rows and exchanges, between them, the work
// vectors lb_opset_phase_exchange lists (all-gather) and the scalar
// (all-reduce); an unsharded apply runs them back to back.
void tmark(lb_opset* h, cudaStream_t st) {
  if (h->timing && h->nev < 16) cudaEventRecord(h->ev[h->nev++], st);
}

// A3 with the fused second sweep (FarA3c + EpiA3p2F, eta from Phi in pass 1):
// exact sweeps only (the FMM path projects its pot/grad/hess outputs onto the
// reference's four quantities) and only once Phi = S^T w has been attached.
bool a3_fused(const lb_opset* h) {
  return h->phi_eta && !h->fmm && h->d.corr[LB_KIND_SPRIME] && h->d.corr[LB_KIND_SPP_PLUS_DPRIME];
}

int apply_phase(lb_opset* h, int form, int phase, const double* tau, double* out, cudaStream_t st) {
  const auto* C = h->d.corr;
  SkLayout L{};
  if (phase == 0) h->nev = 0;
  tmark(h, st);
  if (form == 3) {
    double* s_tau = V(h, 0);
    double* sp_tau = V(h, 1);
    const bool fused = a3_fused(h);
    if (phase == 0) {
      const double* in1[1] = {tau};
      LB_TRY(far_stage(h, FK_A3A, 1, in1, false, &L, st));
      tmark(h, st);
      const double* vals[2] = {C[LB_KIND_S], C[LB_KIND_SPRIME]};
      const double* xs[2] = {tau, tau};
      if (fused) {
        auto e = base_epi<EpiA3p1R>(h, L, 2);
        e.s_tau = s_tau;
        e.sp_tau = sp_tau;
        e.phi = h->phi_eta;  // epilogues index global rows
        return run_csr<2, EpiA3p1R>(h, vals, xs, e, st, h->wsum);
      }
      auto e = base_epi<EpiA3p1>(h, L, 2);
      e.s_tau = s_tau;
      e.sp_tau = sp_tau;
      return run_csr<2, EpiA3p1>(h, vals, xs, e, st);  // MixOneX<2> measured slower (1.39 vs 1.19 ms, config 3)
    }
    if (phase == 1 && fused) {
      const double* in2[2] = {sp_tau, s_tau};  // mu1 = S' tau, mu2 = S tau
      LB_TRY(far_stage(h, FK_A3C, 2, in2, false, &L, st));
      tmark(h, st);
      auto e = base_epi<EpiA3p2F>(h, L, 1);
      e.tau = tau;
      e.curv = h->d.curvature;
      e.eta = h->scal;
      e.result = out;
      const double* vals[3] = {C[LB_KIND_SPRIME], C[LB_KIND_SPRIME], C[LB_KIND_SPP_PLUS_DPRIME]};
      const double* xs[3] = {sp_tau, s_tau, s_tau};
      return run_csr<3, EpiA3p2F, MixA3p2F>(h, vals, xs, e, st);
    }
    if (phase == 2 && fused) return LB_OK;  // eta added by the pass-2 epilogue
    if (phase == 1 && h->fmm && h->fmm_a3_two) {
      // FMM far field: the second call on two densities (X = c0 - dipole c1 n,
      // B = c1) instead of three, projected straight onto the fused sum
      const double* in2[2] = {sp_tau, s_tau};
      LB_TRY(far_stage(h, FK_A3M, 2, in2, false, &L, st));
      tmark(h, st);
      auto e = base_epi<EpiA3p2M>(h, L, 2);
      e.tau = tau;
      e.curv = h->d.curvature;
      e.w = h->d.weights;
      e.result = out;
      const double* vals[4] = {C[LB_KIND_SPRIME], C[LB_KIND_S], C[LB_KIND_SPRIME], C[LB_KIND_SPP_PLUS_DPRIME]};
      const double* xs[4] = {sp_tau, s_tau, s_tau, s_tau};
      return run_csr<4, EpiA3p2M, MixA3p2>(h, vals, xs, e, st, h->wsum);
    }
    if (phase == 1) {
      const double* in2[2] = {sp_tau, s_tau};  // mu1 = S' tau, mu2 = S tau
      LB_TRY(far_stage(h, FK_A3B, 2, in2, false, &L, st));
      tmark(h, st);
      auto e = base_epi<EpiA3p2>(h, L, 4);
      e.tau = tau;
      e.curv = h->d.curvature;
      e.w = h->d.weights;
      e.result = out;
      const double* vals[4] = {C[LB_KIND_SPRIME], C[LB_KIND_S], C[LB_KIND_SPRIME], C[LB_KIND_SPP_PLUS_DPRIME]};
      const double* xs[4] = {sp_tau, s_tau, s_tau, s_tau};
      return run_csr<4, EpiA3p2, MixA3p2>(h, vals, xs, e, st, h->wsum);
    }
    add_scalar_kernel<<<(unsigned)ceil_div(h->nr, 256), 256, 0, st>>>(out + h->r0, h->nr, h->scal);
    LB_CHECK_LAUNCH();
    return LB_OK;
  }
  if (form == 2) {
    double* mu1 = V(h, 0);
    double* mu2 = V(h, 1);
    if (phase == 0) {
      const double* in1[1] = {tau};
      LB_TRY(far_stage(h, FK_A2A, 1, in1, false, &L, st));
      tmark(h, st);
      auto e = base_epi<EpiA2p1>(h, L, 4);
      e.curv = h->d.curvature;
      e.w = h->d.weights;
      e.mu1 = mu1;
      e.mu2 = mu2;
      const double* vals[4] = {C[LB_KIND_S], C[LB_KIND_D], C[LB_KIND_SPRIME], C[LB_KIND_SPP_PLUS_DPRIME]};
      const double* xs[4] = {tau, tau, tau, tau};
      return run_csr<4, EpiA2p1>(h, vals, xs, e, st, h->wsum);
    }
    // mu2 += ws in place (scal[0]) while both are oversampled
    const double* in2[2] = {mu2, mu1};
    LB_TRY(far_stage(h, FK_A2B, 2, in2, true, &L, st));
      tmark(h, st);
    auto e = base_epi<EpiA2p2>(h, L, 2);
    e.tau = tau;
    e.result = out;
    const double* vals[2] = {C[LB_KIND_D], C[LB_KIND_S]};
    const double* xs[2] = {mu1, mu2};
    return run_csr<2>(h, vals, xs, e, st);
  }
  // form == 1
  if (!h->d.tangents_u || !h->d.tangents_v || !h->d.inv_metric || !h->d.phi0)
    return fail(LB_ERR_ARG, "opset: A1 needs tangents, inverse metric and phi0");
  double* mux = V(h, 0);
  double* muy = V(h, 1);
  double* muz = V(h, 2);
  if (phase == 0) {
    const double* in1[1] = {tau};
    LB_TRY(far_stage(h, FK_A1A, 1, in1, false, &L, st));
      tmark(h, st);
    auto e = base_epi<EpiA1p1>(h, L, 4);
    e.tu = h->d.tangents_u;
    e.tv = h->d.tangents_v;
    e.gi = h->d.inv_metric;
    e.w = h->d.weights;
    e.mux = mux;
    e.muy = muy;
    e.muz = muz;
    const double* vals[4] = {C[LB_KIND_S], C[LB_KIND_GRAD_S1], C[LB_KIND_GRAD_S2], C[LB_KIND_GRAD_S3]};
    const double* xs[4] = {tau, tau, tau, tau};
    return run_csr<4, EpiA1p1>(h, vals, xs, e, st, h->wsum);
  }
  const double* in2[3] = {mux, muy, muz};
  LB_TRY(far_stage(h, FK_A1B, 3, in2, false, &L, st));
      tmark(h, st);
  auto e = base_epi<EpiA1p2>(h, L, 1);
  e.phi0 = h->d.phi0;
  e.eta = h->scal;
  e.result = out;
  const double* vals[3] = {C[LB_KIND_GRAD_S1], C[LB_KIND_GRAD_S2], C[LB_KIND_GRAD_S3]};
  const double* xs[3] = {mux, muy, muz};
  return run_csr<3>(h, vals, xs, e, st);
}

int nphases(int form) { return form == 3 ? 3 : 2; }

int apply_layer(lb_opset* h, int kind, const double* tau, double* out, cudaStream_t st) {
  if (kind < 0 || kind >= LB_NKINDS) return fail(LB_ERR_ARG, "opset: unknown kernel kind");
  const double* val = h->d.corr[kind];
  if (!val) return fail(LB_ERR_KEY, "opset: corrections for this kind were not built");
  FarKind fk;
  int nout = 1, o = 0;
  double sign = 1.0;
  switch (kind) {
    case LB_KIND_S: fk = FK_S; break;
    case LB_KIND_SPRIME: fk = FK_A3A; nout = 2; o = 1; sign = -1.0; break;
    case LB_KIND_D: fk = FK_D; break;
    case LB_KIND_SPP_PLUS_DPRIME: fk = FK_A2A; nout = 4; o = 3; break;
    default: fk = FK_A1A; nout = 4; o = 1 + (kind - LB_KIND_GRAD_S1); sign = -1.0; break;
  }
  SkLayout L{};
  const double* in[1] = {tau};
  LB_TRY(far_stage(h, fk, 1, in, false, &L, st));
  auto e = base_epi<EpiLayer>(h, L, nout);
  e.o = o;
  e.sign = sign;
  e.y = out;
  const double* vals[1] = {val};
  const double* xs[1] = {tau};
  return run_csr<1>(h, vals, xs, e, st);
}

// block-CSR index (quadrature.py:693-700: every row is |Near| blocks of nb
// consecutive columns, so one int32 per block carries the pattern): built
// and verified on the device; any row or block that breaks the structure
// (a caller's own CSR) leaves the scalar index in use
__global__ void block_index_kernel(const int64_t* __restrict__ indptr, const int32_t* __restrict__ indices,
                                   int64_t r0, int64_t nr, int nb, int32_t* __restrict__ bstart,
                                   int* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nr) return;
  const int64_t kb = indptr[r0 + i], ke = indptr[r0 + i + 1];
  if (kb % nb || ke % nb) {
    *bad = 1;
    return;
  }
  for (int64_t b = kb / nb; b < ke / nb; ++b) {
    const int32_t c0 = indices[b * nb];
    bstart[b] = c0;
    for (int j = 1; j < nb; ++j)
      if (indices[b * nb + j] != c0 + j) *bad = 1;
  }
}

int build_block_index(lb_opset* h) {
  const int nb = h->d.nb;
  const int64_t nnz = h->d.nnz;
  if (nb <= 1 || nnz <= 0 || nnz % nb) return LB_OK;
  int* bad = nullptr;
  cudaError_t e = cudaMalloc((void**)&h->bstart, sizeof(int32_t) * (nnz / nb));
  if (e == cudaSuccess) e = cudaMalloc((void**)&bad, sizeof(int));
  if (e == cudaSuccess) e = cudaMemset(bad, 0, sizeof(int));
  if (e == cudaSuccess && h->nr > 0) {
    block_index_kernel<<<(unsigned)ceil_div(h->nr, 128), 128>>>(h->d.indptr, h->d.indices, h->r0, h->nr, nb,
                                                                  h->bstart, bad);
    e = cudaGetLastError();
  }
  int hbad = 1;
  if (e == cudaSuccess) e = cudaMemcpy(&hbad, bad, sizeof(int), cudaMemcpyDeviceToHost);
  cudaFree(bad);
  if (e != cudaSuccess) {
    cudaFree(h->bstart);
    h->bstart = nullptr;
    return fail(LB_ERR_CUDA, std::string("lb_opset_create: block index: ") + cudaGetErrorString(e));
  }
  if (hbad) {
    cudaFree(h->bstart);
    h->bstart = nullptr;
  } else {
    h->bnb = nb;
  }
  return LB_OK;
}

}  // namespace
}  // namespace lb

extern "C" {

int lb_opset_create(const lb_opset_desc* d, lb_opset** out) {
  using lb::build_block_index;
  using namespace lb;
  if (!d || !out) return fail(LB_ERR_ARG, "lb_opset_create: null argument");
  *out = nullptr;
  if (d->n <= 0 || d->n_over <= 0 || d->npatches <= 0 || d->nb <= 0 || d->nbo <= 0)
    return fail(LB_ERR_SHAPE, "lb_opset_create: empty discretisation");
  if (d->n != d->npatches * d->nb || d->n_over != d->npatches * d->nbo)
    return fail(LB_ERR_SHAPE, "lb_opset_create: n/n_over do not match npatches*nb/nbo");
  if (!d->nodes || !d->normals || !d->weights || !d->curvature || !d->over_nodes ||
      !d->over_normals || !d->over_weights || !d->over_interp || !d->indptr || !d->indices)
    return fail(LB_ERR_ARG, "lb_opset_create: missing geometry or CSR pattern");
  // nrows < 0: every row; an empty shard is an error (a handle owning no
  // rows would reduce and read rows it never computed)
  if (d->nrows == 0)
    return fail(LB_ERR_SHAPE, "lb_opset_create: empty row range (nrows = 0)");
  if (d->nrows > 0 && (d->row0 < 0 || d->row0 + d->nrows > d->n))
    return fail(LB_ERR_SHAPE, "lb_opset_create: row range outside [0, n)");
  lb_opset* h = new lb_opset();
  h->d = *d;
  h->r0 = d->nrows > 0 ? d->row0 : 0;
  h->nr = d->nrows > 0 ? d->nrows : d->n;
  h->wsum = d->weight_sum;
  const int64_t n = d->n;
  h->ns_pad = ceil_div(d->n_over, kFarPad) * kFarPad;
  int64_t cap = 1;
  cap = std::max(cap, far_part_size<FarS>(h));
  cap = std::max(cap, far_part_size<FarA3a>(h));
  cap = std::max(cap, far_part_size<FarA3b>(h));
  cap = std::max(cap, far_part_size<FarA3c>(h));
  cap = std::max(cap, far_part_size<FarA2a>(h));
  cap = std::max(cap, far_part_size<FarA2b>(h));
  cap = std::max(cap, far_part_size<FarD>(h));
  cap = std::max(cap, far_part_size<FarA1a>(h));
  cap = std::max(cap, far_part_size<FarA1b>(h));
  h->part_cap = cap;
  h->csr_wpr = csr_wpr(d->nnz, n);
  h->csr_blocks = (int)ceil_div(h->nr, (kCsrBT / 32) / h->csr_wpr);
  cudaError_t e = cudaSuccess;
  auto A = [&](void** p, size_t bytes) {
    if (e == cudaSuccess) e = cudaMalloc(p, bytes);
  };
  A((void**)&h->pack4, sizeof(double) * h->ns_pad * 4);
  A((void**)&h->pack6, sizeof(double) * h->ns_pad * 6);
  A((void**)&h->pack8, sizeof(double) * h->ns_pad * 8);
  A((void**)&h->part, sizeof(double) * h->part_cap);
  A((void**)&h->vec, sizeof(double) * n * 8);
  A((void**)&h->partials, sizeof(double) * (h->csr_blocks + 32));
  A((void**)&h->ticket, sizeof(unsigned) * 4);
  A((void**)&h->scal, sizeof(double) * 8);
  if (e == cudaSuccess) e = cudaMemset(h->ticket, 0, sizeof(unsigned) * 4);
  if (e == cudaSuccess) e = cudaMemset(h->scal, 0, sizeof(double) * 8);
  if (e != cudaSuccess) {
    lb_opset_destroy(h);
    return fail(LB_ERR_CUDA, std::string("lb_opset_create: ") + cudaGetErrorString(e));
  }
  const unsigned g = (unsigned)ceil_div(h->ns_pad, 256);
  fill_geom_kernel<<<g, 256>>>(d->over_nodes, nullptr, d->n_over, h->ns_pad, 4, h->pack4);
  fill_geom_kernel<<<g, 256>>>(d->over_nodes, nullptr, d->n_over, h->ns_pad, 6, h->pack6);
  fill_geom_kernel<<<g, 256>>>(d->over_nodes, d->over_normals, d->n_over, h->ns_pad, 8, h->pack8);
  e = cudaGetLastError();
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    lb_opset_destroy(h);
    return fail(LB_ERR_CUDA, std::string("lb_opset_create: ") + cudaGetErrorString(e));
  }
  LB_TRY(build_block_index(h));
  *out = h;
  return LB_OK;
}

int lb_opset_destroy(lb_opset* h) {
  if (!h) return LB_OK;
  cudaFree(h->bstart);
  cudaFree(h->pack4);
  cudaFree(h->pack6);
  cudaFree(h->pack8);
  cudaFree(h->part);
  cudaFree(h->vec);
  cudaFree(h->partials);
  cudaFree(h->ticket);
  cudaFree(h->scal);
  cudaFree(h->f_ch);
  cudaFree(h->f_ch3);
  cudaFree(h->f_dp);
  cudaFree(h->f_pot);
  cudaFree(h->f_grad);
  cudaFree(h->f_hess);
  cudaFree(h->f_proj);
  h->f_proj = nullptr;
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  delete h;
  return LB_OK;
}

int lb_opset_set_fmm(lb_opset* h, lb_fmm_plan* plan) {
  using namespace lb;
  if (!h) return fail(LB_ERR_ARG, "lb_opset_set_fmm: null handle");
  h->fmm = nullptr;
  if (!plan) return LB_OK;
  int64_t sizes[10];
  LB_TRY(lb_fmm_plan_info(plan, sizes, nullptr));
  // targets: this handle's rows, or every node (a replicated plan whose owned
  // target range is this handle's rows, lb_fmm_plan_set_target_range)
  if (sizes[2] != h->d.n_over || (sizes[3] != h->nr && sizes[3] != h->d.n))
    return fail(LB_ERR_SHAPE, "lb_opset_set_fmm: plan sources/targets must be over_nodes/nodes");
  const int64_t no = h->d.n_over, nt = sizes[3];
  if (!h->f_ch || nt > h->fmm_nt) {
    for (double** p : {&h->f_ch, &h->f_ch3, &h->f_dp, &h->f_pot, &h->f_grad, &h->f_hess, &h->f_proj}) {
      cudaFree(*p);
      *p = nullptr;
    }
    cudaError_t e = cudaSuccess;
    auto A = [&](double** p, int64_t k) { if (e == cudaSuccess) e = cudaMalloc((void**)p, sizeof(double) * k); };
    A(&h->f_ch, 3 * no);
    A(&h->f_ch3, 3 * no);
    A(&h->f_dp, 9 * no);
    A(&h->f_pot, 3 * nt);
    A(&h->f_grad, 9 * nt);
    A(&h->f_hess, 27 * nt);
    if (e == cudaSuccess) e = cudaMemset(h->f_ch3, 0, sizeof(double) * 3 * no);
    if (e == cudaSuccess) e = cudaMemset(h->f_dp, 0, sizeof(double) * 9 * no);
    if (e == cudaSuccess) e = cudaMemset(h->f_ch, 0, sizeof(double) * 3 * no);
    if (e != cudaSuccess) return fail(LB_ERR_CUDA, std::string("lb_opset_set_fmm: ") + cudaGetErrorString(e));
  }
  h->fmm_nt = nt;
  // the one-segment projection layout must fit the partial buffer
  const int64_t need = ceil_div(h->nr, 64) * 64 * 4;
  if (need > h->part_cap) {
    cudaFree(h->part);
    h->part = nullptr;
    LB_CUDA(cudaMalloc(&h->part, sizeof(double) * need));
    h->part_cap = need;
  }
  h->fmm = plan;
  return LB_OK;
}

int lb_opset_set_phi0(lb_opset* h, const double* phi0) {
  if (!h) return lb::fail(LB_ERR_ARG, "lb_opset_set_phi0: null handle");
  h->d.phi0 = phi0;
  return LB_OK;
}

int lb_opset_set_fmm_a3(lb_opset* h, int two_densities) {
  if (!h) return lb::fail(LB_ERR_ARG, "lb_opset_set_fmm_a3: null handle");
  h->fmm_a3_two = two_densities != 0;
  return LB_OK;
}

int lb_opset_set_eta_weights(lb_opset* h, const double* phi) {
  if (!h) return lb::fail(LB_ERR_ARG, "lb_opset_set_eta_weights: null handle");
  h->phi_eta = phi;
  return LB_OK;
}

int lb_opset_set_timing(lb_opset* h, int on) {
  if (!h) return lb::fail(LB_ERR_ARG, "lb_opset_set_timing: null handle");
  if (on && !h->ev[0])
    for (auto& e : h->ev) LB_CUDA(cudaEventCreate(&e));
  h->timing = on != 0;
  return LB_OK;
}

// ms between consecutive marks of the last apply: [far 1, csr 1, far 2,
// csr 2 (+ glue)], total in ms[7]
int lb_opset_stage_times(lb_opset* h, double* ms) {
  if (!h || !ms) return lb::fail(LB_ERR_ARG, "lb_opset_stage_times: null argument");
  for (int i = 0; i < 8; ++i) ms[i] = 0.0;
  if (!h->timing || h->nev < 2) return LB_OK;
  LB_CUDA(cudaEventSynchronize(h->ev[h->nev - 1]));
  float t = 0;
  for (int i = 0; i + 1 < h->nev && i < 7; ++i) {
    cudaEventElapsedTime(&t, h->ev[i], h->ev[i + 1]);
    ms[i] = t;
  }
  cudaEventElapsedTime(&t, h->ev[0], h->ev[h->nev - 1]);
  ms[7] = t;
  return LB_OK;
}

int lb_opset_apply(lb_opset* h, int formulation, const double* tau, double* out, void* stream) {
  using namespace lb;
  if (!h || !tau || !out) return fail(LB_ERR_ARG, "lb_opset_apply: null argument");
  if (tau == out) return fail(LB_ERR_ARG, "lb_opset_apply: tau and out must not alias");
  cudaStream_t st = as_stream(stream);
  if (formulation < 1 || formulation > 3)
    return fail(LB_ERR_ARG, "lb_opset_apply: formulation must be 1, 2 or 3");
  if (h->nr != h->d.n)
    return fail(LB_ERR_ARG, "lb_opset_apply: sharded handle; run lb_opset_apply_phase with exchanges");
  for (int p = 0; p < nphases(formulation); ++p) LB_TRY(apply_phase(h, formulation, p, tau, out, st));
  tmark(h, st);
  return LB_OK;
}

int lb_opset_apply_phase(lb_opset* h, int formulation, int phase, const double* tau, double* out,
                         void* stream) {
  using namespace lb;
  if (!h || !tau || !out) return fail(LB_ERR_ARG, "lb_opset_apply_phase: null argument");
  if (formulation < 1 || formulation > 3 || phase < 0 || phase >= nphases(formulation))
    return fail(LB_ERR_ARG, "lb_opset_apply_phase: bad formulation/phase");
  return apply_phase(h, formulation, phase, tau, out, as_stream(stream));
}

int lb_opset_phase_exchange(const lb_opset* h, int formulation, int phase, int* nvec, int* vecs,
                            int* reduce_scalar) {
  using namespace lb;
  if (!h || !nvec || !vecs || !reduce_scalar) return fail(LB_ERR_ARG, "lb_opset_phase_exchange: null");
  *nvec = 0;
  *reduce_scalar = 0;
  if (formulation == 3) {
    // fused A3: eta is reduced by pass 1 (phase 0) and consumed by pass 2
    if (phase == 0) { *nvec = 2; vecs[0] = 0; vecs[1] = 1; *reduce_scalar = a3_fused(h) ? 1 : 0; }
    else if (phase == 1) *reduce_scalar = a3_fused(h) ? 0 : 1;
  } else if (phase == 0) {
    *nvec = formulation == 2 ? 2 : 3;
    for (int k = 0; k < *nvec; ++k) vecs[k] = k;
    *reduce_scalar = 1;
  }
  return LB_OK;
}

int lb_opset_buffers(const lb_opset* h, double** work, double** scalar, int64_t* row0,
                     int64_t* nrows) {
  if (!h) return lb::fail(LB_ERR_ARG, "lb_opset_buffers: null handle");
  if (work) *work = h->vec;
  if (scalar) *scalar = h->scal;
  if (row0) *row0 = h->r0;
  if (nrows) *nrows = h->nr;
  return LB_OK;
}

int lb_opset_apply_layer(lb_opset* h, int kind, const double* tau, double* out, void* stream) {
  using namespace lb;
  if (!h || !tau || !out) return fail(LB_ERR_ARG, "lb_opset_apply_layer: null argument");
  if (tau == out) return fail(LB_ERR_ARG, "lb_opset_apply_layer: tau and out must not alias");
  return apply_layer(h, kind, tau, out, as_stream(stream));
}

int lb_opset_last_scalar(const lb_opset* h, double* dev_out) {
  if (!h || !dev_out) return lb::fail(LB_ERR_ARG, "lb_opset_last_scalar: null argument");
  LB_CUDA(cudaMemcpy(dev_out, h->scal, sizeof(double), cudaMemcpyDeviceToDevice));
  return LB_OK;
}

int lb_opset_time_far(lb_opset* h, int which, int reps, double* seconds_host, void* stream) {
  using namespace lb;
  if (!h || !seconds_host || reps <= 0) return fail(LB_ERR_ARG, "lb_opset_time_far: bad arguments");
  cudaStream_t st = as_stream(stream);
  cudaEvent_t e0, e1;
  LB_CUDA(cudaEventCreate(&e0));
  LB_CUDA(cudaEventCreate(&e1));
  SkLayout ns{};
  int rc = LB_OK;
  LB_CUDA(cudaEventRecord(e0, st));
  for (int r = 0; r < reps && rc == LB_OK; ++r) {
    switch (which) {
      case 0: rc = run_far<FarS>(h, h->pack4, &ns, st); break;
      case 1: rc = run_far<FarA3a>(h, h->pack4, &ns, st); break;
      case 2:
        rc = a3_fused(h) ? run_far<FarA3c>(h, h->pack8, &ns, st) : run_far<FarA3b>(h, h->pack8, &ns, st);
        break;
      case 8: rc = run_far<FarA3b>(h, h->pack8, &ns, st); break;
      case 9: rc = run_far<FarA3c>(h, h->pack8, &ns, st); break;
      case 3: rc = run_far<FarA2a>(h, h->pack8, &ns, st); break;
      case 4: rc = run_far<FarA2b>(h, h->pack8, &ns, st); break;
      case 5: rc = run_far<FarA1a>(h, h->pack4, &ns, st); break;
      case 6: rc = run_far<FarA1b>(h, h->pack6, &ns, st); break;
      case 7: rc = run_far<FarD>(h, h->pack8, &ns, st); break;
      default: rc = fail(LB_ERR_ARG, "lb_opset_time_far: unknown sweep");
    }
  }
  LB_CUDA(cudaEventRecord(e1, st));
  LB_CUDA(cudaEventSynchronize(e1));
  float ms = 0.f;
  LB_CUDA(cudaEventElapsedTime(&ms, e0, e1));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  *seconds_host = (double)ms * 1e-3 / reps;
  return rc;
}

int lb_csr_spmv(const int64_t* indptr, const int32_t* indices, int64_t nrows, int njobs,
                const double* const* vals, const double* const* xs, double* const* ys,
                int accumulate, void* stream) {
  using namespace lb;
  if (njobs < 1 || njobs > 4) return fail(LB_ERR_ARG, "lb_csr_spmv: njobs must be in [1, 4]");
  if (nrows <= 0) return LB_OK;
  cudaStream_t st = as_stream(stream);
  int64_t nnz = 0;
  LB_CUDA(cudaMemcpy(&nnz, indptr + nrows, sizeof(int64_t), cudaMemcpyDeviceToHost));
  const int wpr = csr_wpr(nnz, nrows);
  const unsigned blocks = (unsigned)ceil_div(nrows, (kCsrBT / 32) / wpr);
#define LB_SPMV(J)                                                                          \
  {                                                                                         \
    CsrJobs<J> jobs;                                                                        \
    EpiStore<J> epi;                                                                        \
    for (int j = 0; j < J; ++j) {                                                           \
      jobs.val[j] = vals[j];                                                                \
      jobs.x[j] = xs[j];                                                                    \
      epi.y[j] = ys[j];                                                                     \
    }                                                                                       \
    epi.accumulate = accumulate;                                                            \
    csr_epi_kernel<J, EpiStore<J>, MixId<J>><<<blocks, kCsrBT, 0, st>>>(indptr, indices, nullptr, 0, 0, nrows, wpr, jobs, \
                                                              epi, nullptr, nullptr,        \
                                                              nullptr, 1.0);                \
  }
  switch (njobs) {
    case 1: LB_SPMV(1) break;
    case 2: LB_SPMV(2) break;
    case 3: LB_SPMV(3) break;
    default: LB_SPMV(4) break;
  }
#undef LB_SPMV
  LB_CHECK_LAUNCH();
  return LB_OK;
}

}  // extern "C"
