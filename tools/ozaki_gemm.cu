// Harness for the emulated-fp64 M2L GEMM (tcgen05 kind::i8, Ozaki slicing):
// Y (nrep x ncol, col-major) = A (nrep x nrep, row-major fp64) * X (col-major)
// compared with cuBLAS DGEMM for accuracy and time.  Not part of the library.
#include <cublas_v2.h>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <random>
#include <vector>

#include "../paper_2111_10743_b200/csrc/ozaki.cuh"

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("CUDA %s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

template <int S, int NT = lb::oz::nt_for(S)>
int run(int nrep, int64_t ncol, int reps) {
  using namespace lb::oz;
  const int KC = (nrep + kBK - 1) / kBK, MT = (nrep + kBM - 1) / kBM;
  // kernel-like operator: 1/r between two separated point clouds
  std::mt19937_64 g(7);
  std::uniform_real_distribution<double> U(-1, 1);
  std::vector<double> P(3 * nrep), Q(3 * nrep), A((size_t)nrep * nrep);
  for (int i = 0; i < nrep; ++i)
    for (int a = 0; a < 3; ++a) { P[3 * i + a] = U(g); Q[3 * i + a] = U(g) + (a == 0 ? 4.0 : 0.0); }
  for (int i = 0; i < nrep; ++i)
    for (int j = 0; j < nrep; ++j) {
      double dx = P[3 * i] - Q[3 * j], dy = P[3 * i + 1] - Q[3 * j + 1], dz = P[3 * i + 2] - Q[3 * j + 2];
      A[(size_t)i * nrep + j] = 1.0 / std::sqrt(dx * dx + dy * dy + dz * dz);
    }
  std::normal_distribution<double> N01;
  std::vector<double> X((size_t)nrep * ncol);
  for (auto& x : X) x = N01(g);
  std::vector<uint8_t> Ap((size_t)MT * KC * S * kABytes);
  std::vector<double> rs((size_t)MT * kBM);
  pack_rows_host<S>(A.data(), nrep, Ap.data(), rs.data());
  double *dA, *dX, *dY, *dYr, *drs, *dcs;
  uint8_t *dAp, *dBp;
  const int64_t NTL = (ncol + NT - 1) / NT;
  CK(cudaMalloc(&dA, A.size() * 8));
  CK(cudaMalloc(&dX, X.size() * 8));
  CK(cudaMalloc(&dY, X.size() * 8));
  CK(cudaMalloc(&dYr, X.size() * 8));
  CK(cudaMalloc(&drs, rs.size() * 8));
  CK(cudaMalloc(&dcs, NTL * NT * 8));
  CK(cudaMalloc(&dAp, Ap.size()));
  CK(cudaMalloc(&dBp, (size_t)NTL * KC * S * NT * 32));
  CK(cudaMemcpy(dA, A.data(), A.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dX, X.data(), X.size() * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(dAp, Ap.data(), Ap.size(), cudaMemcpyHostToDevice));
  CK(cudaMemcpy(drs, rs.data(), rs.size() * 8, cudaMemcpyHostToDevice));
  cublasHandle_t h;
  cublasCreate(&h);
  const double one = 1.0, zero = 0.0;
  auto dgemm = [&]() {
    cublasDgemm(h, CUBLAS_OP_T, CUBLAS_OP_N, nrep, (int)ncol, nrep, &one, dA, nrep, dX, nrep, &zero, dYr, nrep);
  };
  auto emu = [&](bool slice, bool mm) {
    if (slice) CK((slice_cols<S, NT>(dX, nrep, nrep, ncol, nullptr, dBp, dcs, 0)));
    if (mm) CK((gemm<S, NT>(dAp, dBp, drs, dcs, nrep, ncol, dY, nrep, 0)));
  };
  dgemm();
  emu(true, true);
  CK(cudaDeviceSynchronize());
  std::vector<double> Y(X.size()), Yr(X.size());
  CK(cudaMemcpy(Y.data(), dY, Y.size() * 8, cudaMemcpyDeviceToHost));
  CK(cudaMemcpy(Yr.data(), dYr, Yr.size() * 8, cudaMemcpyDeviceToHost));
  double emax = 0, ymax = 0, erel = 0;
  for (int64_t c = 0; c < ncol; ++c) {
    double cm = 0, ce = 0;
    for (int r = 0; r < nrep; ++r) {
      cm = std::max(cm, std::fabs(Yr[c * nrep + r]));
      ce = std::max(ce, std::fabs(Y[c * nrep + r] - Yr[c * nrep + r]));
    }
    emax = std::max(emax, ce);
    ymax = std::max(ymax, cm);
    erel = std::max(erel, ce / cm);
  }
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](auto f) {
    for (int i = 0; i < 3; ++i) f();
    cudaEventRecord(e0);
    for (int i = 0; i < reps; ++i) f();
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  const float t_d = timeit(dgemm);
  const float t_s = timeit([&] { emu(true, false); });
  const float t_g = timeit([&] { emu(false, true); });
  const float t_f1 = timeit([&] { CK((gemm<S, NT, 1>(dAp, dBp, drs, dcs, nrep, ncol, dY, nrep, 0))); });
  const float t_f2 = timeit([&] { CK((gemm<S, NT, 2>(dAp, dBp, drs, dcs, nrep, ncol, dY, nrep, 0))); });
  const float t_f3 = timeit([&] { CK((gemm<S, NT, 3>(dAp, dBp, drs, dcs, nrep, ncol, dY, nrep, 0))); });
  const float t_f4 = timeit([&] { CK((gemm<S, NT, 4>(dAp, dBp, drs, dcs, nrep, ncol, dY, nrep, 0))); });
  printf("   no-A-copy %.3f ms  no-B-copy %.3f ms  no-epilogue %.3f ms  no-mma %.3f ms\n", t_f1, t_f2, t_f3, t_f4);
  const double fl = 2.0 * nrep * (double)nrep * ncol;
  const double mma = (double)S * (S + 1) / 2 * 2.0 * MT * kBM * (double)KC * kBK * NTL * NT;
  printf("S=%d NT=%d nrep=%d ncol=%ld | err max %.2e (of %.2e) col-rel %.2e | dgemm %.3f ms (%.1f TF) | "
         "slice %.3f ms | i8gemm %.3f ms (%.1f TF-eq, %.0f TOPS)\n",
         S, NT, nrep, (long)ncol, emax, ymax, erel, t_d, fl / t_d * 1e-9, t_s, t_g, fl / t_g * 1e-9,
         mma / t_g * 1e-9);
  cudaFree(dA); cudaFree(dX); cudaFree(dY); cudaFree(dYr); cudaFree(drs); cudaFree(dcs);
  cudaFree(dAp); cudaFree(dBp);
  cublasDestroy(h);
  return 0;
}

int main(int argc, char** argv) {
  const int64_t ncol = argc > 1 ? atol(argv[1]) : 65536;
  const char* only = argc > 2 ? argv[2] : nullptr;  // e.g. "6" runs only S=6 at nrep 729
  const int reps = 10;
  if (only) {
    switch (atoi(only)) {
      case 4: run<4>(729, ncol, reps); break;
      case 5: run<5>(729, ncol, reps); break;
      case 7: run<7>(729, ncol, reps); break;
      case 6: run<6>(729, ncol, reps); break;
      case 8: run<8>(729, ncol, reps); break;
      default: break;
    }
    return 0;
  }
  run<3>(729, ncol, reps);
  run<4>(729, ncol, reps);
  run<5>(729, ncol, reps);
  run<6>(729, ncol, reps);
  run<7>(729, ncol, reps);
  run<8>(729, ncol, reps);
  run<4>(296, ncol, reps);
  run<5>(296, ncol, reps);
  run<6>(488, ncol, reps);
  run<8>(1331, ncol / 2, reps);
  return 0;
}
