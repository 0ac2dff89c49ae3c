// Tuning harness (not part of the library): fp64 1/r seed + refinement
// variants inside a charge pot+grad P2P loop.  Prints pairs/s, FP64
// instructions are read from `cuobjdump -sass`, and the max relative error of
// pot / |grad| against an IEEE 1/sqrt evaluation of the same sums.
//   make -C tools rsqrt_probe ; ./tools/rsqrt_probe [n]
#include <cuda_runtime.h>
#include <stdint.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

// V0: MUFU.RSQ64H seed + 2nd-order step (5 FP64 ops) — the round-1 kernel
__device__ __forceinline__ double v0(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  y = (__double2hiint(y) == 0x7ff00000) ? 0.0 : y;
  double h = r2 * y;
  double e = fma(-h, y, 1.0);
  double p = fma(e, 0.375, 0.5);
  double q = y * e;
  return fma(q, p, y);
}

// V1: fp32 seed from the top 32 significant bits of r2 (integer rebias, no
// conversion instruction), MUFU.RSQ in fp32, integer back-conversion to fp64
// together with y/2, then ONE Newton step (3 FP64 ops).
__device__ __forceinline__ double v1(double r2) {
  const uint32_t hi = (uint32_t)__double2hiint(r2), lo = (uint32_t)__double2loint(r2);
  // (hi:lo) << 3 keeps exponent bits 8..0 + 23 significand bits; adding
  // 128 << 23 (mod 2^32) turns the fp64 exponent (1024 + k) into fp32 127 + k + 1
  const uint32_t fb = __funnelshift_l(lo, hi, 3) + 0x40000000u;
  float f;
  asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(f) : "f"(__uint_as_float(fb)));
  uint32_t u = __float_as_uint(f);
  const bool zero = hi == 0u;                 // r2 == 0 (or < 2^-1022): skip
  const uint32_t b = zero ? 0u : (896u << 20), bh = zero ? 0u : (895u << 20);
  u = zero ? 0u : u;
  const double y = __hiloint2double((int)((u >> 3) + b), (int)(u << 29));
  const double yh = __hiloint2double((int)((u >> 3) + bh), (int)(u << 29));
  const double e = fma(-r2, y * y, 1.0);
  return fma(yh, e, y);
}

// V2: conversion instructions for the fp32 seed, then one Newton step
__device__ __forceinline__ double v2(double r2) {
  const float f = rsqrtf(__double2float_rn(r2));
  double y = (double)f;
  y = (__double2hiint(r2) == 0) ? 0.0 : y;
  const double e = fma(-r2, y * y, 1.0);
  return fma(0.5 * y, e, y);
}

// V3: MUFU.RSQ64H seed + plain Newton (accuracy reference point only)
__device__ __forceinline__ double v3(double r2) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(r2));
  y = (__double2hiint(y) == 0x7ff00000) ? 0.0 : y;
  const double e = fma(-r2, y * y, 1.0);
  return fma(0.5 * y, e, y);
}

// IEEE reference
__device__ __forceinline__ double vref(double r2) { return r2 == 0.0 ? 0.0 : 1.0 / sqrt(r2); }

template <int V>
__device__ __forceinline__ double isq(double r2) {
  if (V == 0) return v0(r2);
  if (V == 1) return v1(r2);
  if (V == 2) return v2(r2);
  if (V == 3) return v3(r2);
  return vref(r2);
}

template <int V, int TPT, int BT, int TS>
__global__ void __launch_bounds__(BT) p2p(const double4* __restrict__ src, int ns,
                                          const double* __restrict__ tgt, int nt,
                                          double* __restrict__ out) {
  __shared__ double4 sh[TS];
  double tx[TPT], ty[TPT], tz[TPT], a[TPT][4];
#pragma unroll
  for (int j = 0; j < TPT; ++j) {
    const int t = min(nt - 1, (int)(blockIdx.x * BT * TPT + j * BT + threadIdx.x));
    tx[j] = tgt[3 * t];
    ty[j] = tgt[3 * t + 1];
    tz[j] = tgt[3 * t + 2];
    a[j][0] = a[j][1] = a[j][2] = a[j][3] = 0.0;
  }
  for (int s0 = 0; s0 < ns; s0 += TS) {
    __syncthreads();
    for (int k = threadIdx.x; k < TS; k += BT) sh[k] = src[s0 + k];
    __syncthreads();
#pragma unroll 2
    for (int k = 0; k < TS; ++k) {
      const double4 s = sh[k];
#pragma unroll
      for (int j = 0; j < TPT; ++j) {
        const double dx = tx[j] - s.x, dy = ty[j] - s.y, dz = tz[j] - s.z;
        const double rr = fma(dz, dz, fma(dy, dy, dx * dx));
        const double y = isq<V>(rr);
        const double y3 = y * (y * y);
        a[j][0] = fma(s.w, y, a[j][0]);
        const double c3 = s.w * y3;
        a[j][1] = fma(-c3, dx, a[j][1]);
        a[j][2] = fma(-c3, dy, a[j][2]);
        a[j][3] = fma(-c3, dz, a[j][3]);
      }
    }
  }
#pragma unroll
  for (int j = 0; j < TPT; ++j) {
    const int t = blockIdx.x * BT * TPT + j * BT + threadIdx.x;
    if (t < nt)
      for (int c = 0; c < 4; ++c) out[4 * (int64_t)t + c] = a[j][c];
  }
}

template <int V>
double run(const char* name, const double4* src, int ns, const double* tgt, int nt, double* out) {
  constexpr int TPT = 4, BT = 64, TS = 128;
  const int blocks = (nt + BT * TPT - 1) / (BT * TPT);
  for (int w = 0; w < 2; ++w) p2p<V, TPT, BT, TS><<<blocks, BT>>>(src, ns, tgt, nt, out);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int reps = 5;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) p2p<V, TPT, BT, TS><<<blocks, BT>>>(src, ns, tgt, nt, out);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double t = ms / reps * 1e-3;
  const double rate = (double)nt * ns / t;
  printf("%-5s %8.3f ms  %.4e pairs/s  %.2f TF(20flop)\n", name, t * 1e3, rate, rate * 20 / 1e12);
  return rate;
}

int main(int argc, char** argv) {
  const int n = argc > 1 ? atoi(argv[1]) : (1 << 17);
  std::mt19937_64 rng(7);
  std::normal_distribution<double> g;
  std::vector<double> tgt(3 * n);
  std::vector<double> src(4 * n);
  for (int i = 0; i < n; ++i) {
    double x = g(rng), y = g(rng), z = g(rng), r = sqrt(x * x + y * y + z * z);
    tgt[3 * i] = src[4 * i] = x / r;
    tgt[3 * i + 1] = src[4 * i + 1] = y / r;
    tgt[3 * i + 2] = src[4 * i + 2] = z / r;
    src[4 * i + 3] = g(rng);
  }
  double *dt, *ds, *o[5];
  cudaMalloc(&dt, 8 * tgt.size());
  cudaMalloc(&ds, 8 * src.size());
  cudaMemcpy(dt, tgt.data(), 8 * tgt.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(ds, src.data(), 8 * src.size(), cudaMemcpyHostToDevice);
  for (auto& p : o) cudaMalloc(&p, 32 * (size_t)n);
  const double4* s4 = (const double4*)ds;
  run<4>("ieee", s4, n, dt, n, o[4]);
  run<0>("v0", s4, n, dt, n, o[0]);
  run<1>("v1", s4, n, dt, n, o[1]);
  run<2>("v2", s4, n, dt, n, o[2]);
  run<3>("v3", s4, n, dt, n, o[3]);
  std::vector<double> ref(4 * (size_t)n), got(4 * (size_t)n);
  cudaMemcpy(ref.data(), o[4], 32 * (size_t)n, cudaMemcpyDeviceToHost);
  double pmax = 0, gmax = 0;
  for (int i = 0; i < n; ++i) {
    pmax = std::max(pmax, fabs(ref[4 * i]));
    for (int c = 1; c < 4; ++c) gmax = std::max(gmax, fabs(ref[4 * i + c]));
  }
  for (int v = 0; v < 4; ++v) {
    cudaMemcpy(got.data(), o[v], 32 * (size_t)n, cudaMemcpyDeviceToHost);
    double ep = 0, eg = 0;
    for (int i = 0; i < n; ++i) {
      ep = std::max(ep, fabs(got[4 * i] - ref[4 * i]));
      for (int c = 1; c < 4; ++c) eg = std::max(eg, fabs(got[4 * i + c] - ref[4 * i + c]));
    }
    printf("v%d  pot rel err %.3e  grad rel err %.3e\n", v, ep / pmax, eg / gmax);
  }
  // element-wise 1/r accuracy over a log-uniform r2 sweep
  return 0;
}
