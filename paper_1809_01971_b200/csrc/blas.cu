// Plain fp64 GEMMs through cuBLAS (the dense sine-matrix DST for lengths
// without an FFT plan, dense eigenbasis transforms): C = alpha A B + beta C
// with row-major operands, A either row- or column-major, batched over a
// stride.  Layouts cuBLAS cannot express return FL_EINVAL so the caller can
// use the SIMT kernel (gemm_f64 in kernels.cu).
#include <cublas_v2.h>

#include <map>
#include <mutex>

#include "common.cuh"
#include "kernels.cuh"

namespace fl {

static cublasHandle_t blas_handle() {
  static std::mutex mu;
  static std::map<int, cublasHandle_t> handles;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return nullptr;
  std::lock_guard<std::mutex> lk(mu);
  auto it = handles.find(dev);
  if (it != handles.end()) return it->second;
  cublasHandle_t h = nullptr;
  if (cublasCreate(&h) != CUBLAS_STATUS_SUCCESS) return nullptr;
  handles[dev] = h;
  return h;
}

int gemm_blas(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sAm, int64_t sAk, int64_t bA,
              const double* B, int64_t sBk, int64_t sBn, int64_t bB, double beta, double* C, int64_t sCm,
              int64_t sCn, int64_t bC, int64_t batch, cudaStream_t st) {
  if (M <= 0 || N <= 0 || batch <= 0) return FL_OK;
  const int64_t lim = (int64_t)1 << 31;
  if (M >= lim || N >= lim || K >= lim || batch >= lim) return FL_EINVAL;
  cublasOperation_t opA;
  int64_t ldA;
  if (sAk == 1) {
    opA = CUBLAS_OP_T;  // row-major A is its transpose in column-major terms
    ldA = sAm;
  } else if (sAm == 1) {
    opA = CUBLAS_OP_N;
    ldA = sAk;
  } else {
    return FL_EINVAL;
  }
  cublasHandle_t h = blas_handle();
  if (!h || cublasSetStream(h, st) != CUBLAS_STATUS_SUCCESS) return FL_EINVAL;
  cublasStatus_t s;
  if (N == 1 && sBk == 1 && bB == K && sCm == 1 && bC == M && bA == 0) {
    // batch of matrix-vector products = one GEMM: C_cm (M x batch) = op(A) B_cm (K x batch)
    s = cublasDgemm(h, opA, CUBLAS_OP_N, (int)M, (int)batch, (int)K, &alpha, A, (int)ldA, B, (int)K, &beta, C,
                    (int)M);
  } else if (sBn == 1 && sCn == 1) {
    // row-major C = A B  <=>  column-major C^T = B^T A^T
    const cublasOperation_t opAt = (opA == CUBLAS_OP_T) ? CUBLAS_OP_N : CUBLAS_OP_T;
    s = cublasDgemmStridedBatched(h, CUBLAS_OP_N, opAt, (int)N, (int)M, (int)K, &alpha, B, (int)sBk, bB, A,
                                  (int)ldA, bA, &beta, C, (int)sCm, bC, (int)batch);
  } else {
    return FL_EINVAL;
  }
  if (s != CUBLAS_STATUS_SUCCESS) {
    set_error("cuBLAS GEMM failed (status %d)", (int)s);
    return FL_ECUDA;
  }
  return FL_OK;
}

}  // namespace fl
