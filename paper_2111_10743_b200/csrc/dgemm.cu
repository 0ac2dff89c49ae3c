// C-ABI access to the FP64 tensor-core GEMM of the FMM translations
// (dgemm_cols.cuh), for its numerics tests and its roofline probe:
// Y (M x ncols, column-major, ldy) = alpha * A (M x K row-major, lda) * X
// (K x ncols, column-major, ldx), optionally with X's columns gathered
// through cols[] and each column's K index through a permutation table.
#include "dgemm_cols.cuh"
#include "lb_common.cuh"

extern "C" {

int lb_dgemm_cols(const double* A, int lda, int M, int K, const double* X, int64_t ldx,
                  const int64_t* cols, const int32_t* kperm, const int32_t* kp, int64_t ncols,
                  double* Y, int64_t ldy, double alpha, int add, void* stream) {
  using namespace lb;
  if (!A || !X || !Y || M <= 0 || K <= 0 || ncols < 0 || lda < K || ldx < K || ldy < M)
    return fail(LB_ERR_ARG, "lb_dgemm_cols: bad arguments");
  if ((kperm == nullptr) != (kp == nullptr)) return fail(LB_ERR_ARG, "lb_dgemm_cols: kperm needs kp");
  dg::Args a{};
  a.A = A; a.lda = lda; a.M = M; a.K = K; a.S = 1; a.nd = 1;
  a.X = X; a.ldx = ldx; a.in = cols; a.kperm = kperm; a.kp = kp;
  a.Y = Y; a.ldy = ldy; a.alpha = alpha; a.add = add; a.nq = ncols;
  const cudaError_t e = dg::gemm_cols(a, ncols, 1, as_stream(stream));
  if (e != cudaSuccess) return fail(LB_ERR_CUDA, std::string("lb_dgemm_cols: ") + cudaGetErrorString(e));
  return LB_OK;
}

}  // extern "C"
