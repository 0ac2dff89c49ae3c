// Deterministic grid reductions: every block writes one partial, the last
// block to finish (atomic ticket) sums the partials in a fixed order and
// publishes the scalar on the device, then re-arms the ticket.  No host sync,
// no fp64 atomics, bit-identical run to run.
#pragma once

#include "lb_common.cuh"

namespace lb {

template <int BT>
__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x < 32) {
    s = (l < BT / 32) ? sh[l] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  }
  return s;  // valid in warp 0
}

// Called by ALL threads of every block with the block's contribution `v`.
// The last block writes out[0] = op(total).  mode 0: total / div,
// mode 1: sqrt(total).
template <int BT>
__device__ __forceinline__ void grid_reduce_finish(double v, double* partials, unsigned* ticket,
                                                   double* out, int mode, double div) {
  __shared__ double sh[BT / 32];
  __shared__ bool last;
  const double bs = block_sum<BT>(v, sh);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = bs;
    __threadfence();
    const unsigned t = atomicAdd(ticket, 1u);
    last = (t == gridDim.x - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double s = 0.0;
  for (unsigned i = threadIdx.x; i < gridDim.x; i += BT) s += ((volatile double*)partials)[i];
  const double tot = block_sum<BT>(s, sh);
  if (threadIdx.x == 0) {
    out[0] = mode == 1 ? sqrt(tot) : tot / div;
    *ticket = 0u;
  }
}

}  // namespace lb
