/*
 * fraclap_b200 — C ABI of the B200-native hot path of the fractional-Laplacian
 * optimal-control solver (arXiv 1809.01971; reference package `fraclap`).
 *
 * Plain pointers and sizes only: every array argument is a DEVICE pointer to
 * fp64 data (unless stated otherwise), every size is int64_t, `stream` is a
 * cudaStream_t passed as void* (NULL = legacy default stream).  All entry
 * points are asynchronous on `stream` unless marked "sync".
 *
 * Return value: FL_OK (0) on success; FL_EINVAL for an argument the
 * reference would reject with ValueError; FL_ECUDA / FL_ENOMEM for device
 * failures.  fl_last_error() returns the message of the last failure on the
 * calling thread.
 *
 * Layout convention: a d-way full tensor with dims (n0, .., n_{d-1}) is
 * C-ordered (last index fastest).  A canonical factor matrix U^(l) of shape
 * (n_l, R) is row-major (R fastest), exactly the numpy layout of the
 * reference's `CpTensor.factors` (tensor.py:54-96).
 *
 * Reference interface each entry point replaces is cited as file:line of
 * /root/reference/pkg/src/fraclap/.
 */
#ifndef FRACLAP_B200_H
#define FRACLAP_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FL_OK 0
#define FL_EINVAL 1
#define FL_ECUDA 2
#define FL_ENOMEM 3

/* core function tags (fracop.py:58 _TAGS) */
#define FL_G1 0 /* cm * rho^-a                 */
#define FL_G2 1 /* cm * rho^-a + cp * rho^a    */
#define FL_G3 2 /* 1 / g2                      */
#define FL_G4 3 /* 1 / (1 + cp * rho^(2a))     */

/* ---- library / device info ------------------------------------------ */
int fl_version(void);
const char* fl_last_error(void);
int fl_sm_count(void);
/* sync: build the per-n transform tables (twiddles, sine tables, dense sine
 * matrices).  Called implicitly on first use; call it up front before CUDA
 * graph capture. */
int fl_prepare(int64_t n);

/* ---- spectral: orthonormal DST-I --------------------------------------
 * Replaces spectral.dst_apply (spectral.py:163-186, analytic-dst branch:
 * scipy.fft.dst(x, type=1, norm="ortho", axis=0)) and its batched use in
 * fracop.apply (fracop.py:490-493).
 * Treats x as [outer][n][inner] and transforms the middle axis:
 *   y[o][k][c] = scale * sqrt(2/(n+1)) * sum_j sin(pi (j+1)(k+1)/(n+1)) x[o][j][c]
 * x == y (in place) is allowed.  n+1 a power of two in [4, 8192] runs the
 * FFT kernel; any other n runs the dense sine-matrix kernel. */
int fl_dst1(const double* x, double* y, int64_t outer, int64_t n, int64_t inner,
            double scale, void* stream);

/* Fused operator pass along the middle axis: y = scale * F diag(core) F x
 * per line (core in the layout of x).  With inner == 1 this is one kernel
 * (forward DST, core scaling and inverse DST in shared memory); it is the
 * last-mode pass of fl_apply_full. */
int fl_dst1_core(const double* x, double* y, const double* core, int64_t outer, int64_t n,
                 int64_t inner, double scale, void* stream);

/* Dense-eigenbasis transform (spectral.py:184-186 for generalized_mode):
 * y[o] = Q^T x[o] (forward) or Q x[o] (inverse) along the middle axis, Q
 * an (n, n) row-major orthonormal matrix on the device. */
int fl_basis_apply(const double* Q, int transpose, const double* x, double* y,
                   int64_t outer, int64_t n, int64_t inner, void* stream);

/* ---- fracop: cores ------------------------------------------------------
 * Dense core evaluation, fracop._dense_core / _eval_on_rho
 * (fracop.py:109-148): out[i] = g(rho(i)), rho(i) = sum_l mu_l[i_l],
 * with g selected by tag (FL_G1..FL_G4), outer exponent a, coefficients
 * cm, cp, and `reciprocal` (1 -> 1/g).  mu: d device pointers (host array
 * of pointers). */
int fl_core_eval(double* out, int d, const int64_t* dims, const double* const* mu,
                 int tag, double a, double cm, double cp, int reciprocal,
                 void* stream);

/* cp_to_dense (tensor.py:217-225): out[i] = sum_k w[k] prod_l U_l[i_l, k]. */
int fl_cp_to_dense(double* out, int d, const int64_t* dims, int64_t rank,
                   const double* weights, const double* const* factors,
                   void* stream);

/* Sinc-quadrature factors, fracop._sinc_core (fracop.py:194-199):
 * U[i, k] = exp(-(mu[i] / rho_min) * t[k]) for an (n, R) row-major U. */
int fl_sinc_factor(double* U, const double* mu, int64_t n, const double* t,
                   int64_t R, double rho_min, void* stream);

/* ---- full-format operator application ---------------------------------
 * y = alpha * F diag(core) F x on a d-way tensor (d = 2 or 3), F the
 * per-mode orthonormal DST-I (the full-format form of fracop.apply; the
 * reference's dense oracle is tests/oracles.py:56 dense_apply).  `core` is
 * a dense core tensor of the same dims (from fl_core_eval / fl_cp_to_dense).
 * x == y allowed.  The last mode runs forward DST, core scaling and the
 * inverse DST in one fused pass; the other modes one pass each way. */
int fl_apply_full(const double* x, double* y, const double* core, int d,
                  const int64_t* dims, double alpha, void* stream);

/* Same operator on a padded internal layout: the last mode's rows have
 * pitch `pitch` >= n_last (e.g. 512 for n = 511) so every row starts on a
 * 128-byte boundary.  core_p is the core in that padded layout; work is a
 * caller-owned padded buffer (prod(dims[:-1]) * pitch doubles, padding
 * zero-initialised once).  x and y are dense (unpadded); the first pass
 * reads x into the padded layout and the last writes y back, so the
 * intermediate passes run on aligned rows.  All modes must be FFT lengths
 * (n+1 a power of two).  x == y allowed. */
int fl_apply_full_padded(const double* x, double* y, const double* core_p, double* work,
                         int d, const int64_t* dims, int64_t pitch, double alpha,
                         void* stream);

/* Same operator for n_0 = n_last = 511 (N = 512, the configs[2] grid)
 * through the register-resident passes: last mode first (contiguous dense
 * rows into the padded work tensor), mode 1, then mode 0 forward + core +
 * inverse in one pass, mode 1, last mode back into y.  core_l is the core
 * in the mode-0 lane order read by the fused pass with one coalesced
 * 512-byte load per warp instruction: with G padded to [511][n1][512]
 * (pad column zero; n1 = 1 for d = 2), unit u = (i1 * 32 + c) * 4 + w
 * covers columns i2 = 16c + 4w .. 16c + 4w + 3; entry ((u * 32 + i) * 32
 * + 16 f + q) is the double pair (G[r - 1][i1][16c + 4w + 2f],
 * G[r - 1][i1][16c + 4w + 2f + 1]), r = 32q + i (r = 0 gives zeros).
 * work: [511][n1][512] doubles, padding zero-initialised once. */
int fl_apply_full_lanes(const double* x, double* y, const double* core_l, double* work,
                        int d, const int64_t* dims, double alpha, void* stream);

/* The fused mode-0 pass of fl_apply_full_lanes on its own (per-pass timing):
 * y = scale * F_0 diag(core_l) F_0 x on [511][groups][512], x == y allowed. */
int fl_dst1_core_lanes_mode0(const double* x, double* y, const double* core_l, int64_t groups,
                             double scale, void* stream);

/* Fused pass along contiguous lines with a line-ordered core (n = 511):
 * `lines` lines of pitch `pitch` (>= 512, even), y = scale * F diag(G) F x
 * per line; core_l is G in the line lane order: unit u = lines 4u .. 4u+3,
 * entry ((u * 32 + i) * 32 + 16 f + q) = (G[4u + 2f][r - 1],
 * G[4u + 2f + 1][r - 1]), r = 32q + i, units padded to a multiple of 4.
 * x == y allowed. */
int fl_dst1_core_lanes(const double* x, double* y, const double* core_l, int64_t lines,
                       int64_t pitch, double scale, void* stream);

/* One DST-I pass with explicit layouts (the building block of the two
 * calls above; exposed for per-pass timing).  contig != 0: `outer` lines,
 * row j of line L at L*lp + j.  contig == 0: `outer` blocks of `groups`
 * column groups of `width` columns, element (block o, group g, column c,
 * row j) at o*os + g*gp + c + j*js.  in_layout / out_layout are int64[4]
 * {os, js, gp, lp} for x (and core) / y.  core != NULL (contig only) runs
 * the fused forward-scale-inverse pass.  FFT lengths only.  `contig` is a
 * flag word: FL_PASS_CONTIG selects contiguous lines; FL_PASS_PAD_WRITE
 * lets a strided pass with an odd width write the column after each group
 * (the padding of an internal work buffer, as in fl_apply_full_padded)
 * so that it can store 16-byte line pairs, and makes a contiguous pass with
 * out pitch > n zero the padding of every line (later strided passes pair
 * the last column with the padding in one packed FFT, so it must hold a
 * defined value); without it the padding is never written. */
#define FL_PASS_CONTIG 1
#define FL_PASS_PAD_WRITE 2
int fl_dst1_pass(const double* x, double* y, const double* core, int64_t n, int contig,
                 int64_t outer, int64_t groups, int64_t width, const int64_t* in_layout,
                 const int64_t* out_layout, double scale, void* stream);

/* y = alpha * F x over all d modes (a full spectral transform). */
int fl_transform_full(const double* x, double* y, int d, const int64_t* dims,
                      double alpha, void* stream);

/* ---- canonical format --------------------------------------------------
 * One mode of the canonical operator application, fracop.apply
 * (fracop.py:474-495): out (n, R*S) with column k*S + s equal to
 * scale * F(U[:, k] .* Xs[:, s]); U is the (n, R) core factor, Xs the
 * already transformed (n, S) operand factor.  The Hadamard expansion is
 * formed while loading the DST tile (no n x R*S intermediate). */
int fl_cp_apply_mode(const double* U, const double* Xs, double* out, int64_t n,
                     int64_t R, int64_t S, double scale, void* stream);

/* Hadamard product of per-mode Gram matrices, the kernel of cp_inner
 * (tensor.py:156-167): H[i][j] = prod_l sum_r A_l[r][i] B_l[r][j] for d
 * factor pairs A_l (n_l, Ra), B_l (n_l, Rb); H is (Ra, Rb) row-major. */
int fl_cp_gram(int d, const int64_t* n, const double* const* A, int64_t Ra,
               const double* const* B, int64_t Rb, double* H, void* stream);

/* Batched thin SVD of small matrices (one-sided Jacobi, one CTA per
 * matrix): A is batch x m x n row-major; U (batch, m, k), S (batch, k)
 * descending, Vt (batch, k, n), k = min(m, n).  The slice SVDs of t2c
 * (decomp.py:468-519).  Working set in shared memory up to m = n = 110,
 * beyond that in a device scratch allocated on the stream.  Vt may be NULL
 * when m >= n: left vectors and values only (no right rotations are
 * accumulated), e.g. the square R factors of _left_sv. */
int fl_svd_batched(const double* A, int batch, int m, int n, double* U, double* S,
                   double* Vt, void* stream);

/* Left singular system of T = A^T for a batch of square k x k matrices A
 * (row-major, k <= 128): a column-pivoted Householder QR of A in shared
 * memory (R only), then one-sided Jacobi on R^T (Drmac-Veselic
 * preconditioning); U (batch, k, k) = left singular vectors of T, S (batch,
 * k) decreasing.  Used by the truncation's factor SVDs after an R-only QR of
 * the long side (decomp._left_sv; reference decomp.py:343-345, 395). */
int fl_svd_left_pivoted(const double* A, int batch, int k, double* U, double* S, void* stream);

/* Khatri-Rao contraction on the FP64 tensor cores (hand-written DMMA GEMM
 * whose A operand is generated while loading, reduction split over R with a
 * fixed-order second pass): out[(ia, ib), j] = sum_r Pa[ia, r] Pb[ib, r]
 * Y[r, j].  Pa (a x R) and Pb (b x R) row-major contiguous; Y element (r, j)
 * at Y[r * sYr + j * sYj]; out (a*b x N) row-major contiguous.  The ALS
 * matrices U_l (KR(Pa, Pb) diag(xi))^T of canonical-to-Tucker and the core
 * projection (decomp.py:349-353, 384-399). */
int fl_kr_contract(const double* Pa, int64_t a, const double* Pb, int64_t b, int64_t R,
                   const double* Y, int64_t sYr, int64_t sYj, int64_t N, double* out,
                   void* stream);

/* Limits of the batched wide-matrix factorisations below. */
#define FL_QR_MAX_BATCH 8
#define FL_QR_MAX_K 128
#define FL_QR_MAX_LEAVES 256

/* R factors of tall-skinny QR factorisations, hand-written TSQR (Householder
 * leaves in shared memory, pairwise merges of the triangles): for each of
 * batch <= FL_QR_MAX_BATCH wide matrices M_i (k_i x m_i, 1 <= k_i <=
 * FL_QR_MAX_K, element (r, c) at M_i[r * rs_i + c * cs_i], one of the two
 * strides equal to 1 for coalesced reads) R_i (k_i x k_i row-major, upper
 * triangular, zeros below) with M_i^T = Q R_i.  M, k, m, rs, cs, R are host
 * arrays of length batch.  Replaces the library geqrf in the truncation's
 * factor SVDs (decomp.py:343-345, 373, 395) and in the range finder. */
int fl_qr_r(int batch, const double* const* M, const int* k, const int64_t* m,
            const int64_t* rs, const int64_t* cs, double* const* R, void* stream);

/* Left singular systems of the same kind of batch: fl_qr_r followed by the
 * pivoted one-CTA Jacobi of fl_svd_left_pivoted on every R_i^T, all matrices
 * in one launch each (the three mode factors of rhosvd / _pick_ranks,
 * decomp.py:343-345, 373, run concurrently).  U_i (k_i x k_i row-major,
 * columns = left singular vectors of M_i) and S_i (k_i, decreasing); U may be
 * NULL, or hold NULL entries, for singular values only. */
int fl_left_sv_wide(int batch, const double* const* M, const int* k, const int64_t* m,
                    const int64_t* rs, const int64_t* cs, double* const* U,
                    double* const* S, void* stream);

/* Column norms of an (n, R) matrix (cp_normalize, tensor.py:180-197). */
int fl_col_norms(const double* U, int64_t n, int64_t R, double* out, void* stream);

/* V = U with columns divided by nrm; zero columns become e_1
 * (tensor.py:189-195). */
int fl_col_scale(const double* U, const double* nrm, int64_t n, int64_t R,
                 double* V, void* stream);

/* ---- full-format PCG (solver.py:116-180 on dense tensors) --------------
 * Spectral-space PCG for the operator F diag(A) F with preconditioner
 * F diag(P) F: b_hat = F b is the transformed right-hand side, x_hat the
 * transformed solution (x = F x_hat); r and p are N-double work arrays.
 * The whole solve is ONE cooperative persistent launch: no host round trip
 * per iteration; one streaming pass (64 B/DoF) and one grid barrier per
 * iteration.  hist (device, k_max + 1 doubles) receives the relative
 * residual history ||r_k|| / ||b||; status (device, 4 ints) receives
 * [iterations, converged, breakdown iteration, breakdown kind (1: <R,Z> <= 0,
 * 2: <P,S> <= 0)], the reference's PcgBreakdownError conditions; on a
 * breakdown hist[breakdown iteration] holds the offending inner product. */
int fl_pcg_spectral(const double* b_hat, double* x_hat, double* r, double* p,
                    const double* A, const double* P, int64_t N, double tol,
                    int k_max, double* hist, int* status, void* stream);

#define FL_PCG_WORK 8192
/* One streaming pass of the same iteration for the slab-partitioned
 * multi-GPU solve (the caller all-reduces the 4 sums in `out` across ranks):
 *   phase 0: x = 0, r = b, p = 0;
 *            out = [b.b, <b, P b>, <P b, A P b>, 0]
 *   phase 1: p = P r + beta p, x += alpha p, r -= alpha A p, z = P r;
 *            out = [r.r, <r, z>, <z, A z>, <z, A p>]
 * (the reference iteration with <P,S> of the next direction from
 * <z,Az> + 2 beta' <z,Ap> + beta'^2 <p,Ap>, see fl_pcg_spectral).
 * work: FL_PCG_WORK doubles zeroed once before the first call. */
int fl_pcg_phase(int phase, const double* b_hat, double* x_hat, double* r, double* p,
                 const double* A, const double* P, int64_t N, double alpha, double beta,
                 double* out, double* work, void* stream);

#ifdef __cplusplus
}
#endif

#endif /* FRACLAP_B200_H */
