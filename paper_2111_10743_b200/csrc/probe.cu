// Hardware probes used by bench.py / tests to state rooflines from measured
// numbers: an FP64 FMA-pipe peak kernel and a dump of the MUFU.RSQ64H seed
// (its accuracy decides how many refinement steps inv_sqrt_skip needs).
#include "lb_common.cuh"

namespace lb {

// 8 independent DFMA chains per thread; each iteration = 8 DFMA = 16 flop
__global__ void __launch_bounds__(256) dfma_peak_kernel(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  double s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  if (s == 12345.678) out[blockIdx.x] = s;  // keep the chains alive
}

// FP64 tensor-core (DMMA 8x8x4) peak: 8 independent accumulator tiles per
// warp; each mma = 8*8*4 FMA = 512 flop per warp
__device__ __forceinline__ void dmma_884(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__global__ void __launch_bounds__(256) dmma_peak_kernel(double* out, int iters, double a) {
  double c[8][2];
#pragma unroll
  for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = threadIdx.x * 1e-3 + t;
  double av = a + threadIdx.x * 1e-9, bv = a - threadIdx.x * 1e-9;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) dmma_884(c[t][0], c[t][1], av, bv);
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

// operand-delivery variants of the DMMA peak probe: MODE 1 changes the A
// fragment register with every DMMA (B fixed), MODE 2 changes both -- a real
// GEMM's inner loop (the peak kernel above feeds every DMMA the same A / B)
template <int MODE>
__global__ void __launch_bounds__(256) dmma_operand_kernel(double* out, int iters, double a) {
  double c[8][2], av[8], bv[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    c[t][0] = c[t][1] = threadIdx.x * 1e-3 + t;
    av[t] = a + (threadIdx.x + t) * 1e-9;
    bv[t] = a - (threadIdx.x + 3 * t) * 1e-9;
  }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int t = 0; t < 8; ++t) dmma_884(c[t][0], c[t][1], av[t], MODE == 2 ? bv[t] : bv[0]);
  }
  double s = 0.0;
#pragma unroll
  for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  if (s == 12345.678) out[blockIdx.x] = s;
}

// do the FP64 tensor cores and the FP64 FMA pipe run side by side?  warps
// 0..NW_MMA-1 of the block run DMMA chains, the rest DFMA chains (iteration
// counts separate, either may be 0); compare the time with each half alone
__global__ void __launch_bounds__(256) mixed_peak_kernel(double* out, int it_mma, int it_fma,
                                                          int nw_mma, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double s = 0.0;
  if (warp < nw_mma) {
    double c[8][2];
#pragma unroll
    for (int t = 0; t < 8; ++t) c[t][0] = c[t][1] = threadIdx.x * 1e-3 + t;
    double av = a + threadIdx.x * 1e-9, bv = a - threadIdx.x * 1e-9;
    for (int i = 0; i < it_mma; ++i) {
#pragma unroll
      for (int t = 0; t < 8; ++t) dmma_884(c[t][0], c[t][1], av, bv);
    }
#pragma unroll
    for (int t = 0; t < 8; ++t) s += c[t][0] + c[t][1];
  } else {
    double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
    for (int i = 0; i < it_fma; ++i) {
#pragma unroll
      for (int k = 0; k < 16; ++k) {
        x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
        x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
      }
    }
    s = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
  }
  if (s == 12345.678) out[blockIdx.x] = s;
}

// HBM read ceiling for the correction SpMV's access shape: one warp per
// "row" of rowlen doubles in each of two streams, 256-byte warp loads, eight
// in flight per stream and lane, rows dealt to 8-warp blocks as csr_epi_kernel
// deals them; no index, no gather, no epilogue
__global__ void __launch_bounds__(256) read_rows_kernel(const double* __restrict__ a,
                                                         const double* __restrict__ b, int64_t nrows,
                                                         int64_t rowlen, double* __restrict__ out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t row = (int64_t)blockIdx.x * 8 + warp;
  if (row >= nrows) return;
  const int64_t kb = row * rowlen, ke = kb + rowlen;
  double s0 = 0.0, s1 = 0.0;
  int64_t k = kb + lane;
  for (; k + 7 * 32 < ke; k += 8 * 32) {
    double va[8], vb[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) va[u] = __ldg(a + k + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) vb[u] = __ldg(b + k + 32 * u);
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      s0 += va[u];
      s1 += vb[u];
    }
  }
  for (; k < ke; k += 32) {
    s0 += __ldg(a + k);
    s1 += __ldg(b + k);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    s0 += __shfl_xor_sync(0xffffffffu, s0, o);
    s1 += __shfl_xor_sync(0xffffffffu, s1, o);
  }
  if (lane == 0) out[row] = s0 + s1;
}

__global__ void rsqrt_seed_kernel(const double* x, double* y, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = rsqrt_seed(x[i]);
}

__global__ void inv_sqrt_kernel(const double* x, double* y, int64_t n) {
  int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) y[i] = inv_sqrt_skip(x[i]);
}

}  // namespace lb

extern "C" {

// flops executed = blocks * 256 * iters * 16 * 8 * 2
int lb_probe_dfma(double* scratch, int blocks, int iters, void* stream) {
  lb::dfma_peak_kernel<<<blocks, 256, 0, lb::as_stream(stream)>>>(scratch, iters, 0.999999, 1e-7);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// flops executed = blocks * 8 warps * iters * 8 mma * 512
int lb_probe_dmma(double* scratch, int blocks, int iters, void* stream) {
  lb::dmma_peak_kernel<<<blocks, 256, 0, lb::as_stream(stream)>>>(scratch, iters, 1e-3);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// as lb_probe_dmma with a different A fragment (mode 1) or A and B fragment
// (mode 2) register per DMMA
int lb_probe_dmma_operands(double* scratch, int blocks, int iters, int mode, void* stream) {
  if (mode == 1) lb::dmma_operand_kernel<1><<<blocks, 256, 0, lb::as_stream(stream)>>>(scratch, iters, 1e-3);
  else lb::dmma_operand_kernel<2><<<blocks, 256, 0, lb::as_stream(stream)>>>(scratch, iters, 1e-3);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// DMMA flops = blocks * nw_mma * it_mma * 8 * 512; DFMA flops = blocks * (8 - nw_mma) * 32 * it_fma * 256
int lb_probe_mixed(double* scratch, int blocks, int it_mma, int it_fma, int nw_mma, void* stream) {
  lb::mixed_peak_kernel<<<blocks, 256, 0, lb::as_stream(stream)>>>(scratch, it_mma, it_fma, nw_mma,
                                                                    0.999999, 1e-7);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// bytes read = 2 * nrows * rowlen * 8
int lb_probe_read_rows(const double* a, const double* b, int64_t nrows, int64_t rowlen, double* out,
                       void* stream) {
  if (nrows <= 0) return LB_OK;
  lb::read_rows_kernel<<<(unsigned)lb::ceil_div(nrows, 8), 256, 0, lb::as_stream(stream)>>>(a, b, nrows, rowlen, out);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

// mode 0: raw MUFU.RSQ64H seed; mode 1: refined inv_sqrt_skip
int lb_probe_rsqrt(const double* x, double* y, int64_t n, int mode, void* stream) {
  if (n <= 0) return LB_OK;
  unsigned g = (unsigned)lb::ceil_div(n, 256);
  if (mode == 0)
    lb::rsqrt_seed_kernel<<<g, 256, 0, lb::as_stream(stream)>>>(x, y, n);
  else
    lb::inv_sqrt_kernel<<<g, 256, 0, lb::as_stream(stream)>>>(x, y, n);
  LB_CHECK_LAUNCH();
  return LB_OK;
}

}  // extern "C"
