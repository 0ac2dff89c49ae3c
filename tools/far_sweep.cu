// Tuning harness (not part of the library): times opfar_kernel variants
// (functor x targets-per-thread x split policy) on a config-2-sized random
// sphere problem.  Build: make -C tools far_sweep ; run on the GPU box.
#include <string>
#include <cstdio>
#include <cstdlib>
#include <random>
#include <vector>

#include "../paper_2111_10743_b200/csrc/opfar.cuh"

using namespace lb;

namespace lb {
static thread_local std::string g_err;
void set_error(const std::string& m) { g_err = m; }
int fail(int c, const std::string& m) { g_err = m; return c; }
int sm_count() { int n = 0; cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, 0); return n; }
}  // namespace lb

template <class F, int TPT, int BT, int TS = 128, bool PF = true, int UR = 2, int MINB = 1>
void run(const char* name, const double* nodes, const double* normals, int64_t n, const double* pack,
         int64_t ns_pad, double* part, int grid_mult) {
  auto kern = opfar_kernel<F, TPT, BT, TS, PF, UR, MINB>;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, BT, 0);
  const SkLayout L = make_sk_layout(n, ns_pad, BT * TPT, TS, (int64_t)sm_count() * per_sm * grid_mult);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 3; ++w) kern<<<(unsigned)L.G, BT>>>(nodes, normals, n, pack, L, part, nodes);
  const int reps = 20;
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) kern<<<(unsigned)L.G, BT>>>(nodes, normals, n, pack, L, part, nodes);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  const double t = ms / reps * 1e-3;
  const double pairs = (double)n * (ns_pad);
  int regs = 0;
  cudaFuncAttributes fa;
  if (cudaFuncGetAttributes(&fa, kern) == cudaSuccess) regs = fa.numRegs;
  printf("%-8s UR=%d MINB=%d regs=%d PF=%d TS=%d TPT=%d BT=%d gridx%d per_sm=%d G=%lld kmax=%lld  %.1f us  %.3e pairs/s\n", name, UR, MINB, regs, (int)PF, TS, TPT, BT,
         grid_mult, per_sm, (long long)L.G, (long long)L.kmax, t * 1e6, pairs / t);
}

int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 8960;
  const int64_t ns = argc > 2 ? atoll(argv[2]) : 35840;
  const int64_t ns_pad = ceil_div(ns, 128) * 128;
  std::mt19937_64 rng(5);
  std::normal_distribution<double> g;
  std::vector<double> nodes(3 * n), normals(3 * n), pack(8 * ns_pad, 0.0);
  for (int64_t i = 0; i < n; ++i) {
    double x = g(rng), y = g(rng), z = g(rng), r = sqrt(x * x + y * y + z * z);
    nodes[3 * i] = normals[3 * i] = x / r;
    nodes[3 * i + 1] = normals[3 * i + 1] = y / r;
    nodes[3 * i + 2] = normals[3 * i + 2] = z / r;
  }
  for (int64_t i = 0; i < ns; ++i) {
    double x = g(rng), y = g(rng), z = g(rng), r = sqrt(x * x + y * y + z * z);
    double* p = &pack[8 * i];
    p[0] = p[3] = x / r; p[1] = p[4] = y / r; p[2] = p[5] = z / r;
    p[6] = g(rng) * 1e-4; p[7] = g(rng) * 1e-4;
  }
  double *dn, *dnn, *dp, *dpart;
  cudaMalloc(&dn, 8 * 3 * n);
  cudaMalloc(&dnn, 8 * 3 * n);
  cudaMalloc(&dp, 8 * 8 * ns_pad);
  cudaMalloc(&dpart, (size_t)8 * 4 * (n + 1024) * 4200);
  cudaMemcpy(dn, nodes.data(), 8 * 3 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dnn, normals.data(), 8 * 3 * n, cudaMemcpyHostToDevice);
  cudaMemcpy(dp, pack.data(), 8 * 8 * ns_pad, cudaMemcpyHostToDevice);
  // A3 call 2 uses the 8-double record; A3 call 1 reads the first 4 doubles
  // of a 4-double record: reuse the buffer (layout-only timing)
  const bool only_a3a = argc > 3 && std::string(argv[3]) == "a3a";
  for (int w : {1}) {
    if (only_a3a) {
      for (int rep = 0; rep < 2; ++rep) {
        run<FarA3c, 2, 64, 128, true, 4, 1>("A3c*", dn, dnn, n, dp, ns_pad, dpart, w);  // shipped
        run<FarA3c, 2, 64, 64, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
        run<FarA3c, 2, 64, 64, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
        run<FarA3c, 3, 64, 64, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
        run<FarA3c, 1, 128, 64, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
        run<FarA3c, 2, 64, 32, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
        run<FarA3c, 2, 64, 64, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, 2);
        run<FarA3c, 1, 64, 64, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
      }
      continue;
    }
    run<FarA1a, 4, 64, 64, true, 2, 1>("A1a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA1a, 2, 64, 128, true, 4, 1>("A1a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA1a, 3, 64, 128, true, 2, 1>("A1a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 2, 64, 128, true, 2, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 2, 64, 128, true, 4, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 128, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 128, true, 2, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 3, 64, 128, true, 2, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 4, 64, 128, true, 2, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 64, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 128, 128, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 128, true, 8, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 256, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 1, 128, 128, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 128, false, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 128, true, 4, 2>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 32, 128, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3c, 2, 64, 128, true, 4, 1>("A3c", dn, dnn, n, dp, ns_pad, dpart, 2);
    run<FarA3b, 2, 64, 128, true, 1, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 2, 64, 128, false, 2, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 2, 64, 128, false, 2, 12>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 2, 128, 128, true, 2, 5>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 3, 64, 128, true, 2, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 1, 128, 128, false, 4, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3b, 1, 256, 128, false, 2, 1>("A3b", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 4, 64, 64, true, 2, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 4, 64, 128, true, 2, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 2, 64, 128, true, 4, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 3, 64, 128, true, 2, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 4, 64, 64, true, 4, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 4, 64, 64, true, 1, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 4, 64, 64, false, 2, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 2, 128, 64, false, 2, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 2, 64, 64, false, 4, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
    run<FarA3a, 6, 64, 64, true, 2, 1>("A3a", dn, dnn, n, dp, ns_pad, dpart, w);
  }
  cudaError_t e = cudaDeviceSynchronize();
  printf("status %s\n", cudaGetErrorString(e));
  return e != cudaSuccess;
}
