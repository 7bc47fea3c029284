// Internal (C++) entry points shared between the translation units.
#pragma once

#include "common.cuh"

namespace fl {

int prepare(int64_t n);

// one side of a DST pass layout (see DstArgs in dst_fft.cuh)
struct PassLayout {
  int64_t os, js, gp, lp;
};

bool fft_length(int64_t n);

int svd_batched(const double* A, int batch, int m, int n, double* U, double* S, double* Vt, cudaStream_t st);
int svd_left_pivoted(const double* A, int batch, int k, double* U, double* S, cudaStream_t st);
int tsqr_r(int batch, const double* const* M, const int* k, const int64_t* m, const int64_t* rs, const int64_t* cs,
           double* const* R, cudaStream_t st);
int left_sv_wide(int batch, const double* const* M, const int* k, const int64_t* m, const int64_t* rs,
                 const int64_t* cs, double* const* U, double* const* S, cudaStream_t st);

int dst_pass(const double* x, double* y, const double* core, int64_t n, bool contig, int64_t outer, int64_t groups,
             int64_t wv, const PassLayout& in, const PassLayout& out, double scale, cudaStream_t st,
             bool pad_write = false);

// fused forward / core / inverse pass, n = 511, lane-ordered core (dst_reg.cuh)
int dst_pass_lanes(const double* x, double* y, const double* core_l, int64_t lines, int64_t pitch, double scale,
                   cudaStream_t st);

// the same along mode 0 of a padded [511][groups][512] tensor (strided tiles),
// core in the mode-0 lane order (fl_apply_full_lanes)
int dst_pass_lanes_mode0(const double* x, double* y, const double* core_l, int64_t groups, double scale,
                         cudaStream_t st);

// y = scale * F x along the middle axis of [outer][n][inner]; with core != nullptr
// y = scale * F diag(core) F x (core in the layout of x)
int dst_mode(const double* x, double* y, int64_t outer, int64_t n, int64_t inner, double scale,
             const double* core, cudaStream_t st);

// out[:, k*S + s] = scale * F(U[:, k] .* Xs[:, s])
int dst_kr(const double* U, const double* Xs, double* out, int64_t n, int64_t R, int64_t S, double scale,
           cudaStream_t st);

// C[b] = alpha * A[b] B[b] (.* E[b]) + beta * C[b] with arbitrary element
// strides, FP64 tensor cores (gemm_dmma.cu); E (optional) shares C's strides
int gemm_f64_ep(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sAm, int64_t sAk,
                int64_t bA, const double* B, int64_t sBk, int64_t sBn, int64_t bB, double beta, double* C,
                int64_t sCm, int64_t sCn, int64_t bC, int64_t batch, const double* E, cudaStream_t st);
int gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sAm, int64_t sAk,
             int64_t bA, const double* B, int64_t sBk, int64_t sBn, int64_t bB, double beta, double* C,
             int64_t sCm, int64_t sCn, int64_t bC, int64_t batch, cudaStream_t st);

// out[(ia, ib), j] = sum_r Pa[ia, r] Pb[ib, r] Y[r, j] (kr_contract.cu); Pa (a x R), Pb (b x R) row-major,
// Y element (r, j) at Y[r * sYr + j * sYj], out (a b x N) row-major
int kr_contract(const double* Pa, int64_t a, const double* Pb, int64_t b, int64_t R, const double* Y, int64_t sYr,
                int64_t sYj, int64_t N, double* out, cudaStream_t st);

int ew_mul(const double* a, const double* b, double* out, int64_t count, double scale, cudaStream_t st);

int kr_expand(const double* U, const double* Xs, double* out, int64_t n, int64_t R, int64_t S, cudaStream_t st);

int core_eval(double* out, int d, const int64_t* dims, const double* const* mu, int tag, double a, double cm,
              double cp, int recip, cudaStream_t st);

int cp_to_dense(double* out, int d, const int64_t* dims, int64_t R, const double* w, const double* const* U,
                cudaStream_t st);

int gram_hadamard(int d, const int64_t* n, const double* const* A, int64_t Ra, const double* const* B, int64_t Rb,
                  double* H, cudaStream_t st);

int col_norms(const double* U, int64_t n, int64_t R, double* out, cudaStream_t st);

int col_scale(const double* U, const double* nrm, int64_t n, int64_t R, double* V, cudaStream_t st);

int pcg_spectral(const double* b, double* x, double* r, double* p, const double* A, const double* P, int64_t N,
                 double tol, int kmax, double* hist, int* status, cudaStream_t st);

int pcg_phase(int which, const double* b, double* x, double* r, double* p, const double* A, const double* P,
              int64_t N, double alpha, double beta, double* out, double* work, cudaStream_t st);

int sinc_factor(double* U, const double* mu, int64_t n, const double* t, int64_t R, double rho_min,
                cudaStream_t st);

}  // namespace fl
