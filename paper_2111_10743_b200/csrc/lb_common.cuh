// Shared plumbing for libb200lb: status codes, last-error string, stream-
// ordered scratch, launch helpers and the fp64 inverse-square-root used by
// every pairwise kernel.  sm_100a only.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cmath>
#include <string>

#include "../../include/lapbel_b200.h"

namespace lb {

// ---------------------------------------------------------------------------
// error handling: every C-ABI entry point returns an lb_status and leaves a
// human-readable message behind for lb_last_error_string().

void set_error(const std::string& msg);
int fail(int code, const std::string& msg);

#define LB_CUDA(expr)                                                        \
  do {                                                                       \
    cudaError_t _e = (expr);                                                 \
    if (_e != cudaSuccess)                                                   \
      return ::lb::fail(LB_ERR_CUDA, std::string(#expr) + ": " +            \
                                         cudaGetErrorString(_e));            \
  } while (0)

#define LB_CHECK_LAUNCH()                                                    \
  do {                                                                       \
    cudaError_t _e = cudaGetLastError();                                     \
    if (_e != cudaSuccess)                                                   \
      return ::lb::fail(LB_ERR_CUDA, std::string("kernel launch (") +       \
                                         __FILE__ + ":" +                    \
                                         std::to_string(__LINE__) + "): " +  \
                                         cudaGetErrorString(_e));            \
  } while (0)

#define LB_TRY(expr)                                                         \
  do {                                                                       \
    int _s = (expr);                                                         \
    if (_s != LB_OK) return _s;                                              \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Stream-ordered scratch that is released on the same stream when it goes out
// of scope (cudaMallocAsync pool: no device-wide sync, reuse across calls).
struct Scratch {
  void* ptr = nullptr;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(const Scratch&) = delete;
  Scratch& operator=(const Scratch&) = delete;
  int alloc(size_t bytes, cudaStream_t s) {
    stream = s;
    if (bytes == 0) bytes = 16;
    cudaError_t e = cudaMallocAsync(&ptr, bytes, s);
    if (e != cudaSuccess) {
      ptr = nullptr;
      return fail(LB_ERR_CUDA, std::string("cudaMallocAsync: ") + cudaGetErrorString(e));
    }
    return LB_OK;
  }
  template <class T> T* as() const { return reinterpret_cast<T*>(ptr); }
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
};

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------------------
// fp64 1/sqrt(r2) with the coincident-pair skip of fmm.py:136-141 /
// _pointsum.py:41-42 folded in (returns 0 when r2 == 0).
//
// Seed: MUFU.RSQ64H (rsqrt.approx.ftz.f64, ~2^-22 relative) on the MUFU pipe,
// off the FP64 pipe.  Refinement: one 2nd-order step
//     e = 1 - r2 y^2,   y <- y (1 + e/2 + 3e^2/8)
// whose truncation error is O(e^3) ~ 2^-66, i.e. below fp64 rounding: 5 FP64
// ops (DMUL, DFMA, DFMA, DMUL, DFMA).  A zero seed stays zero through the
// refinement (e = 1, y = 0), so skipping costs only a select.
__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

__device__ __forceinline__ double inv_sqrt_skip(double r2) {
  double y = rsqrt_seed(r2);
  // r2 == 0 (or an ftz-flushed denormal, r < 1.5e-154) seeds +inf: test the
  // seed's high word on the integer pipe instead of a DSETP on the FP64 pipe
  y = (__double2hiint(y) == 0x7ff00000) ? 0.0 : y;
  double h = r2 * y;
  double e = fma(-h, y, 1.0);
  double p = fma(e, 0.375, 0.5);
  double q = y * e;
  return fma(q, p, y);
}

}  // namespace lb
