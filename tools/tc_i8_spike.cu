// Feasibility spike (not part of the library; A_TMEM variant: A read from TMEM): one CTA computes
// C[128 x N] (int32) = A[128 x K] . B[N x K]^T with tcgen05.mma kind::i8,
// operands K-major in the SWIZZLE_NONE (interleaved core-matrix) layout,
// accumulator in TMEM, read back with tcgen05.ld.  Checked against the host.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("CUDA %s at %d: %s\n", #x, __LINE__, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

// smem matrix descriptor, SWIZZLE_NONE, K-major: LBO = stride between the two
// 16-byte K chunks of one MMA-K, SBO = stride between 8-row groups (bytes)
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= (uint64_t)((saddr >> 4) & 0x3FFF);
  d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
  d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
  d |= (uint64_t)1 << 46;  // version 1 (sm100)
  // base offset 0, lbo mode 0, layout type 0 = SWIZZLE_NONE
  return d;
}

// instruction descriptor: S32 accum, s8 x s8, K-major both, N, M=128
__host__ __device__ constexpr uint32_t make_idesc_i8(int M, int N) {
  return (2u << 4)            // c_format S32
         | (1u << 7)          // a_format signed 8
         | (1u << 10)         // b_format signed 8
         | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

template <int N, int ATM>
__global__ void __launch_bounds__(128) spike_kernel(const int8_t* A, const int8_t* B, int K, int32_t* C) {
  constexpr int M = 128;
  extern __shared__ __align__(1024) uint8_t smem[];
  // layout: [ks][group][chunk][row][16]
  const int KS = K / 32;
  uint8_t* sA = smem;
  uint8_t* sB = smem + KS * (M / 8) * 256;
  __shared__ uint64_t mbar;
  __shared__ uint32_t tmem_base;
  const int tid = threadIdx.x;
  for (int idx = tid; idx < M * K; idx += blockDim.x) {
    const int m = idx / K, k = idx % K;
    sA[(k / 32) * (M / 8) * 256 + (m / 8) * 256 + ((k % 32) / 16) * 128 + (m % 8) * 16 + (k % 16)] = A[m * K + k];
  }
  for (int idx = tid; idx < N * K; idx += blockDim.x) {
    const int n = idx / K, k = idx % K;
    sB[(k / 32) * (N / 8) * 256 + (n / 8) * 256 + ((k % 32) / 16) * 128 + (n % 8) * 16 + (k % 16)] = B[n * K + k];
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&mbar)));
  }
  if (tid < 32) {  // warp 0 allocates TMEM: 512 columns (acc at 0, A at 256)
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;");  // smem writes -> async (tensor) proxy
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = tmem_base;
  const uint32_t tmA = tmem + 256;
  if (ATM == 2) {
    // tcgen05.cp smem (canonical K-major core matrices) -> TMEM, issued in order with the MMAs
    if (tid == 0)
      for (int ks = 0; ks < KS && ks < 32; ++ks)
        asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(tmA + 8 * ks),
                     "l"(make_desc(smem_u32(sA + ks * (M / 8) * 256), 128, 256)));
  }
  if (ATM == 1) {
    // row tid of A, K chunk ks -> TMEM lane tid, columns 8 ks .. 8 ks + 7 (4 int8 per column)
    const int w = tid / 32;
    for (int ks = 0; ks < KS && ks < 32; ++ks) {
      uint32_t r[8];
      for (int c = 0; c < 8; ++c) {
        uint32_t v = 0;
        for (int b = 0; b < 4; ++b) v |= (uint32_t)(uint8_t)A[tid * K + ks * 32 + 4 * c + b] << (8 * b);
        r[c] = v;
      }
      asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"r"(
                       tmA + ((uint32_t)(w * 32) << 16) + (uint32_t)(8 * ks)),
                   "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]));
    }
    asm volatile("tcgen05.wait::st.sync.aligned;");
    asm volatile("tcgen05.fence::before_thread_sync;");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;");
  }
  if (tid == 0) {
    const uint32_t idesc = make_idesc_i8(M, N);
    for (int ks = 0; ks < KS; ++ks) {
      const uint64_t da = make_desc(smem_u32(sA + ks * (M / 8) * 256), 128, 256);
      const uint64_t db = make_desc(smem_u32(sB + ks * (N / 8) * 256), 128, 256);
      const uint32_t acc = ks > 0 ? 1u : 0u;
      if (ATM)
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], [%1], %2, %3, p;\n\t}\n" ::"r"(tmem),
            "r"(tmA + 8 * ks), "l"(db), "r"(idesc), "r"(acc));
      else
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}\n" ::"r"(tmem),
            "l"(da), "l"(db), "r"(idesc), "r"(acc));
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
        smem_u32(&mbar)));
  }
  // wait for the MMAs (bounded spin: never hang the box)
  {
    uint32_t done = 0;
    for (int it = 0; it < (1 << 24) && !done; ++it) {
      asm volatile(
          "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0, 1, 0, p;\n\t}\n"
          : "=r"(done)
          : "r"(smem_u32(&mbar)), "r"(0));
    }
    if (!done) asm volatile("trap;");
  }
  asm volatile("tcgen05.fence::after_thread_sync;");
  // warp w reads TMEM lanes [32w, 32w+32): one row per thread, 8 columns per load
  const int warp = tid / 32, lane = tid % 32;
  const int row = warp * 32 + lane;
  for (int c0 = 0; c0 < N; c0 += 8) {
    uint32_t v[8];
    const uint32_t taddr = tmem + ((uint32_t)(warp * 32) << 16) + (uint32_t)c0;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
                 : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
                   "=r"(v[7])
                 : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;");
    for (int j = 0; j < 8; ++j) C[row * N + c0 + j] = (int32_t)v[j];
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (tid < 32)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512));
}

template <int N, int ATM = 0>
int run(int K) {
  const int M = 128;
  std::vector<int8_t> A(M * K), B(N * K);
  srand(1);
  for (auto& a : A) a = (int8_t)(rand() % 255 - 127);
  for (auto& b : B) b = (int8_t)(rand() % 255 - 127);
  int8_t *dA, *dB;
  int32_t* dC;
  CK(cudaMalloc(&dA, A.size()));
  CK(cudaMalloc(&dB, B.size()));
  CK(cudaMalloc(&dC, 4 * M * N));
  CK(cudaMemcpy(dA, A.data(), A.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dB, B.data(), B.size(), cudaMemcpyHostToDevice));
  const size_t sm = (size_t)(M + N) * K;
  CK(cudaFuncSetAttribute(spike_kernel<N, ATM>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  spike_kernel<N, ATM><<<1, 128, sm>>>(dA, dB, K, dC);
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  std::vector<int32_t> C(M * N);
  CK(cudaMemcpy(C.data(), dC, 4 * M * N, cudaMemcpyDeviceToHost));
  long bad = 0;
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      long s = 0;
      for (int k = 0; k < K; ++k) s += (long)A[m * K + k] * B[n * K + k];
      if (s != C[m * N + n]) {
        if (bad < 5) printf("  mismatch m=%d n=%d got %d want %ld\n", m, n, C[m * N + n], s);
        ++bad;
      }
    }
  printf("N=%d K=%d A_in_tmem=%d mismatches=%ld\n", N, K, (int)ATM, bad);
  cudaFree(dA); cudaFree(dB); cudaFree(dC);
  return bad != 0;
}

int main() {
  int rc = 0;
  rc |= run<64>(64);
  rc |= run<64>(128);
  rc |= run<128>(320);
  rc |= run<256>(96);
  rc |= run<64, 1>(64);
  rc |= run<128, 1>(320);
  rc |= run<64, 2>(64);
  rc |= run<128, 2>(320);
  printf("%s\n", rc ? "FAIL" : "PASS");
  return rc;
}
