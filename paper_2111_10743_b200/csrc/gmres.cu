// GMRES vector kernels (solver.py:48-103): modified Gram-Schmidt Arnoldi with
// every dot product fused into the preceding axpy's pass over v, norms and
// normalisation, and the final basis combination.  All scalars stay on the
// device (deterministic last-block reductions, reduce.cuh); the host reads
// one Hessenberg column per iteration for the Givens update, as the
// reference's convergence test requires.
#include <algorithm>
#include <map>
#include <mutex>
#include <utility>

#include "lb_common.cuh"
#include "reduce.cuh"

namespace lb {

constexpr int kVecBT = 256;

struct RedBufs {
  double* partials;
  unsigned* ticket;
};

// one pass over i:  v -= hp * qp (if qp), then block-sum of (qn . v) or (v . v)
//   mode 0: out = sum(qn * v)         (MGS dot with the next basis row)
//   mode 1: out = sqrt(sum(v * v))    (the Arnoldi norm)
__global__ void __launch_bounds__(kVecBT) mgs_pass_kernel(double* __restrict__ v,
                                                          const double* __restrict__ qp,
                                                          const double* __restrict__ hp,
                                                          const double* __restrict__ qn,
                                                          int64_t n, int mode, double* out,
                                                          RedBufs rb) {
  const double hv = qp ? hp[0] : 0.0;
  double s = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * kVecBT + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * kVecBT) {
    double x = v[i];
    if (qp) {
      x = fma(-hv, qp[i], x);
      v[i] = x;
    }
    s = fma(mode == 0 ? qn[i] : x, x, s);
  }
  grid_reduce_finish<kVecBT>(s, rb.partials, rb.ticket, out, mode, 1.0);
}

__global__ void scale_inv_kernel(const double* __restrict__ x, const double* __restrict__ s,
                                 int64_t n, double* __restrict__ y) {
  const double d = s[0];
  if (d == 0.0) return;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] = x[i] / d;
}

__global__ void combine_rows_kernel(const double* __restrict__ Q, int64_t ldq, int k, int64_t n,
                                    const double* __restrict__ y, double* __restrict__ x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int j = 0; j < k; ++j) s = fma(y[j], Q[(int64_t)j * ldq + i], s);
    x[i] = s;
  }
}

// Small-N Arnoldi step in ONE CTA: v lives in registers for the whole MGS
// sweep (k+1 dots/axpys + norm + normalise in one launch instead of k+3
// latency-bound grid passes).  Used for n <= kSmallN (config 2: n = 8960).
constexpr int kSmallBT = 1024;
constexpr int64_t kSmallN = 12288;  // 12 doubles of v per thread, in registers

__device__ __forceinline__ double cta_sum(double v, double* red) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (w == 0) {
    s = l < (int)(blockDim.x >> 5) ? red[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (l == 0) red[32] = s;
  }
  __syncthreads();
  return red[32];
}

__global__ void __launch_bounds__(kSmallBT) mgs_small_kernel(double* __restrict__ Q, int64_t ldq, int k,
                                                             int n, double* __restrict__ v,
                                                             double* __restrict__ h) {
  // each thread owns elements threadIdx.x + e*kSmallBT, e < kPer, kept in
  // registers; every basis row is loaded with all kPer loads in flight
  constexpr int kPer = (int)(kSmallN / kSmallBT);
  __shared__ double red[33];
  double x[kPer];
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int i = threadIdx.x + e * kSmallBT;
    x[e] = i < n ? v[i] : 0.0;
  }
  for (int j = 0; j <= k; ++j) {
    const double* q = Q + (int64_t)j * ldq;
    double s = 0.0;
#pragma unroll
    for (int e0 = 0; e0 < kPer; e0 += 4) {  // 4 loads in flight per chunk
      double qv[4];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int i = threadIdx.x + (e0 + e) * kSmallBT;
        qv[e] = i < n ? q[i] : 0.0;
      }
#pragma unroll
      for (int e = 0; e < 4; ++e) s = fma(qv[e], x[e0 + e], s);
    }
    const double hj = cta_sum(s, red);
    if (threadIdx.x == 0) h[j] = hj;
#pragma unroll
    for (int e = 0; e < kPer; ++e) {  // second read of Q_j hits L1
      const int i = threadIdx.x + e * kSmallBT;
      if (i < n) x[e] = fma(-hj, q[i], x[e]);
    }
  }
  double s = 0.0;
#pragma unroll
  for (int e = 0; e < kPer; ++e) s = fma(x[e], x[e], s);
  const double nrm = sqrt(cta_sum(s, red));
  if (threadIdx.x == 0) h[k + 1] = nrm;
  double* qn = Q + (int64_t)(k + 1) * ldq;
#pragma unroll
  for (int e = 0; e < kPer; ++e) {
    const int i = threadIdx.x + e * kSmallBT;
    if (i < n) {
      v[i] = x[e];
      if (nrm != 0.0) qn[i] = x[e] / nrm;
    }
  }
}

namespace {

// persistent reduction scratch, one pool per (device, stream): the grid
// reductions count finished CTAs on a ticket, so two reductions in flight on
// different streams (or devices) must never share partials or tickets.
// Calls on ONE stream are ordered by the stream and share its pool.  A stream
// being captured into a CUDA graph cannot allocate: it borrows the pool of
// the device's first stream (a captured graph replays on its own stream, and
// replays of graphs that share a pool must not overlap).
struct RedPool {
  double* partials = nullptr;
  unsigned* ticket = nullptr;
  int cap = 0;
};

int get_pool(RedBufs* rb, int blocks, cudaStream_t st) {
  static std::mutex mu;
  static std::map<std::pair<int, cudaStream_t>, RedPool> pools;
  static std::map<int, std::pair<int, cudaStream_t>> first;
  int dev = 0;
  LB_CUDA(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lock(mu);
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  LB_CUDA(cudaStreamIsCapturing(st, &cs));
  auto key = std::make_pair(dev, st);
  if (cs != cudaStreamCaptureStatusNone && !pools.count(key)) {
    auto f = first.find(dev);
    if (f == first.end() || pools[f->second].cap < blocks)
      return fail(LB_ERR_CUDA, "reduction scratch: run one reduction on this device before capturing a graph");
    key = f->second;
  }
  RedPool& pool = pools[key];
  if (!first.count(dev)) first[dev] = key;
  if (pool.cap < blocks) {
    if (pool.partials) cudaFree(pool.partials);
    if (pool.ticket) cudaFree(pool.ticket);
    pool.partials = nullptr;
    pool.ticket = nullptr;
    pool.cap = 0;
    LB_CUDA(cudaMalloc(&pool.partials, sizeof(double) * (blocks + 32)));
    LB_CUDA(cudaMalloc(&pool.ticket, sizeof(unsigned) * 4));
    LB_CUDA(cudaMemset(pool.ticket, 0, sizeof(unsigned) * 4));
    pool.cap = blocks;
  }
  rb->partials = pool.partials;
  rb->ticket = pool.ticket;
  return LB_OK;
}

int vec_blocks(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(n, kVecBT * 4), 2 * (int64_t)sm_count()));
}

}  // namespace
}  // namespace lb

extern "C" {

int lb_arnoldi_mgs(double* Q, int64_t ldq, int k, int64_t n, double* v, double* h, void* stream) {
  using namespace lb;
  if (!Q || !v || !h || k < 0 || n <= 0 || ldq < n) return fail(LB_ERR_ARG, "lb_arnoldi_mgs: bad arguments");
  cudaStream_t st = as_stream(stream);
  if (n <= kSmallN) {
    mgs_small_kernel<<<1, kSmallBT, 0, st>>>(Q, ldq, k, (int)n, v, h);
    LB_CHECK_LAUNCH();
    return LB_OK;
  }
  const int blocks = vec_blocks(n);
  RedBufs rb;
  LB_TRY(get_pool(&rb, 2 * sm_count() + 8, st));
  // h[0] = Q_0 . v ; then for j >= 1: v -= h[j-1] Q_{j-1} fused with h[j] = Q_j . v
  for (int j = 0; j <= k; ++j) {
    const double* qp = j > 0 ? Q + (int64_t)(j - 1) * ldq : nullptr;
    mgs_pass_kernel<<<blocks, kVecBT, 0, st>>>(v, qp, j > 0 ? h + j - 1 : nullptr,
                                               Q + (int64_t)j * ldq, n, 0, h + j, rb);
    LB_CHECK_LAUNCH();
  }
  // v -= h[k] Q_k fused with ||v||
  mgs_pass_kernel<<<blocks, kVecBT, 0, st>>>(v, Q + (int64_t)k * ldq, h + k, nullptr, n, 1,
                                             h + k + 1, rb);
  LB_CHECK_LAUNCH();
  scale_inv_kernel<<<blocks, kVecBT, 0, st>>>(v, h + k + 1, n, Q + (int64_t)(k + 1) * ldq);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

int lb_combine_rows(const double* Q, int64_t ldq, int k, int64_t n, const double* y, double* x,
                    void* stream) {
  using namespace lb;
  if (n <= 0) return LB_OK;
  combine_rows_kernel<<<vec_blocks(n), kVecBT, 0, as_stream(stream)>>>(Q, ldq, k, n, y, x);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

int lb_dot(const double* x, const double* y, int64_t n, double* out, void* stream) {
  using namespace lb;
  RedBufs rb;
  LB_TRY(get_pool(&rb, 2 * sm_count() + 8, as_stream(stream)));
  // v := x is read-only here (qp == nullptr), so the const_cast is never written through
  mgs_pass_kernel<<<vec_blocks(std::max<int64_t>(n, 1)), kVecBT, 0, as_stream(stream)>>>(
      const_cast<double*>(x), nullptr, nullptr, y, n, 0, out, rb);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

int lb_nrm2(const double* x, int64_t n, double* out, void* stream) {
  using namespace lb;
  RedBufs rb;
  LB_TRY(get_pool(&rb, 2 * sm_count() + 8, as_stream(stream)));
  mgs_pass_kernel<<<vec_blocks(std::max<int64_t>(n, 1)), kVecBT, 0, as_stream(stream)>>>(
      const_cast<double*>(x), nullptr, nullptr, nullptr, n, 1, out, rb);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

int lb_scale_inv(const double* x, const double* s, int64_t n, double* y, void* stream) {
  using namespace lb;
  if (n <= 0) return LB_OK;
  scale_inv_kernel<<<vec_blocks(n), kVecBT, 0, as_stream(stream)>>>(x, s, n, y);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

}  // extern "C"
