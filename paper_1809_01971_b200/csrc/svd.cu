// Batched SVD of small dense matrices by one-sided (Hestenes) Jacobi, one CTA
// per matrix, the matrix and the accumulated right rotations resident in
// shared memory.  Used by t2c (decomp.py:468-519: one SVD per core slice),
// where the library's batched routines either loop over the batch (gesvd,
// gesvdj beyond 32 x 32) or are approximate (gesvda).
//
// Columns of W (m x n, m >= n; the transpose is processed when m < n) are
// orthogonalised pairwise: a round-robin ordering gives n/2 disjoint pairs
// per round, one warp per pair; a rotation zeroes the pair's inner product.
// Sweeps repeat until no pair has |a_p . a_q| > tol sqrt(|a_p|^2 |a_q|^2).
// Then sigma_j = |a_j|, u_j = a_j / sigma_j, V = accumulated rotations;
// outputs are sorted by decreasing sigma.
#include <atomic>
#include <cstdlib>
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

namespace {

constexpr int SVD_THREADS = 1024;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// players 0..N-1 (N even): round r pairs 0 with pos(0) and pos(k) with
// pos(N-1-k), pos(i) = 1 + (i + r) mod (N - 1)
__device__ __forceinline__ void rr_pair(int N, int r, int k, int& p, int& q) {
  // i + r < 2 (N - 1): one conditional subtraction instead of a modulo
  auto pos = [&](int i) {
    const int x = i + r;
    return 1 + (x >= N - 1 ? x - (N - 1) : x);
  };
  if (k == 0) {
    p = 0;
    q = pos(0);
  } else {
    p = pos(k);
    q = pos(N - 1 - k);
  }
}

// A: batch of m x n row-major matrices (leading dim n, batch stride m*n).
// Outputs: U (batch, m, k), S (batch, k), Vt (batch, k, n), k = min(m, n).
// Placement: W and V in shared memory when both fit, else V (and if need be
// W) in a global scratch buffer (scratch != nullptr; per matrix gstride =
// M*K + (Vt ? K*K : 0) doubles), which stays L2-resident for the sizes of t2c.  Vt == nullptr
// (m >= n only): left vectors and values only, no V is accumulated.
__global__ void __launch_bounds__(SVD_THREADS) k_svd_jacobi(const double* __restrict__ A, int m, int n,
                                                            double* __restrict__ U, double* __restrict__ S,
                                                            double* __restrict__ Vt, int max_sweeps,
                                                            double* scratch, size_t gstride, int w_in_smem,
                                                            int v_in_smem) {
  extern __shared__ double sm_svd[];
  const bool tr = m < n;
  const int M = tr ? n : m;  // rows of the working matrix W
  const int K = tr ? m : n;  // columns of W (= number of singular values)
  const int N = K + (K & 1);
  const bool want_v = Vt != nullptr;
  double* gs = scratch ? scratch + (size_t)blockIdx.x * gstride : nullptr;
  double* sp = sm_svd;
  double* W = w_in_smem ? sp : gs;  // column-major M x K
  if (w_in_smem) sp += (size_t)M * K;
  double* V = !want_v ? nullptr : v_in_smem ? sp : gs + (size_t)M * K;  // column-major K x K
  if (want_v && v_in_smem) sp += (size_t)K * K;
  int* flag = reinterpret_cast<int*>(sp);
  const double* Ab = A + (size_t)blockIdx.x * m * n;
  // load W = A (columns of A) or A^T (rows of A) column-major
  for (int idx = threadIdx.x; idx < m * n; idx += blockDim.x) {
    const int i = idx / n, j = idx - i * n;  // A[i][j]
    if (!tr)
      W[(size_t)j * M + i] = Ab[idx];
    else
      W[(size_t)i * M + j] = Ab[idx];
  }
  if (want_v)
    for (int idx = threadIdx.x; idx < K * K; idx += blockDim.x) V[idx] = (idx / K == idx % K) ? 1.0 : 0.0;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const double tol = 1e-15 * (double)M;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      for (int k = warp; k < N / 2; k += nwarps) {
        int p, q;
        rr_pair(N, r, k, p, q);
        if (p >= K || q >= K) continue;
        double* wp = W + (size_t)p * M;
        double* wq = W + (size_t)q * M;
        double al = 0.0, be = 0.0, ga = 0.0;
        for (int i = lane; i < M; i += 32) {
          const double x = wp[i], y = wq[i];
          al = fma(x, x, al);
          be = fma(y, y, be);
          ga = fma(x, y, ga);
        }
        al = warp_sum(al);
        be = warp_sum(be);
        ga = warp_sum(ga);
        if (fabs(ga) <= tol * sqrt(al * be) || ga == 0.0) continue;
        if (lane == 0) *flag = 1;
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
        const double c = 1.0 / sqrt(1.0 + t * t), s = c * t;
        for (int i = lane; i < M; i += 32) {
          const double x = wp[i], y = wq[i];
          wp[i] = c * x - s * y;
          wq[i] = s * x + c * y;
        }
        if (!want_v) continue;
        double* vp = V + (size_t)p * K;
        double* vq = V + (size_t)q * K;
        for (int i = lane; i < K; i += 32) {
          const double x = vp[i], y = vq[i];
          vp[i] = c * x - s * y;
          vq[i] = s * x + c * y;
        }
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
    if (!any) break;
  }
  // singular values = column norms; rank by decreasing sigma (ties by index)
  double* sig = reinterpret_cast<double*>(flag + 2);  // K doubles after the flag
  for (int j = warp; j < K; j += nwarps) {
    const double* wj = W + (size_t)j * M;
    double a = 0.0;
    for (int i = lane; i < M; i += 32) a = fma(wj[i], wj[i], a);
    a = warp_sum(a);
    if (lane == 0) sig[j] = sqrt(a);
  }
  __syncthreads();
  double* Ub = U + (size_t)blockIdx.x * m * K;
  double* Sb = S + (size_t)blockIdx.x * K;
  double* Vb = want_v ? Vt + (size_t)blockIdx.x * K * n : nullptr;
  for (int j = warp; j < K; j += nwarps) {
    const double sj = sig[j];
    int rank = 0;
    for (int i = lane; i < K; i += 32) rank += (sig[i] > sj || (sig[i] == sj && i < j)) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (lane == 0) Sb[rank] = sj;
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    const double* wj = W + (size_t)j * M;
    const double* vj = want_v ? V + (size_t)j * K : nullptr;
    if (!tr) {
      // A = W_final V^T: U[:, rank] = w_j / s_j (m rows), Vt[rank, :] = v_j (n = K)
      for (int i = lane; i < m; i += 32) Ub[(size_t)i * K + rank] = (sj > 0.0) ? wj[i] * inv : (i == j ? 1.0 : 0.0);
      if (want_v)
        for (int i = lane; i < n; i += 32) Vb[(size_t)rank * n + i] = vj[i];
    } else {
      // A^T = W V^T -> A = V W^T: U[:, rank] = v_j (m = K rows), Vt[rank, :] = w_j / s_j
      for (int i = lane; i < m; i += 32) Ub[(size_t)i * K + rank] = vj[i];
      for (int i = lane; i < n; i += 32) Vb[(size_t)rank * n + i] = (sj > 0.0) ? wj[i] * inv : (i == j ? 1.0 : 0.0);
    }
  }
}

// Small-matrix fast path (m, n <= 128, m >= n, left vectors only): the
// shapes of the truncation's factor SVDs after the QR reduction (127 x 127
// for configs[1]).  Same one-sided Jacobi and the same convergence rule as
// k_svd_jacobi, mapped for issue efficiency: JS_LPP (8) lanes per column
// pair (each lane holds ROWS / 8 rows of both columns as 16-byte pairs), so
// one warp runs 4 pairs and a round of all n/2 pairs is up to 16 warps; the
// per-pair scalar work (reductions, rotation) is shared by 8 lanes instead
// of 32.  (Four lanes per pair, 8 warps: the rounds are latency-bound and
// ran ~1.4x longer, tools/jsmall_var.py.)  The
// working matrix is column-major in shared memory (rows zero-padded to 128,
// column stride 130 doubles to spread the 8 columns a warp touches over the
// banks); the rotation test is done on squares (no square root).
#ifndef FL_JS_LPP
#define FL_JS_LPP 8
#endif
// LPP lanes per column pair; 64 pairs (128 columns) per round
constexpr int JS_ROWS = 128, JS_LPP = FL_JS_LPP, JS_THREADS = 64 * JS_LPP;

// ROWS: working rows (m <= ROWS, zero-padded), 32 / 64 / 128 -> each lane
// holds ROWS / 4 rows of both columns of its pair.
// PIV (square input A, m == n): the left singular system of T = A^T with the
// Drmac-Veselic preconditioning: a column-pivoted Householder QR A P = Q R
// in shared memory (R only), then one-sided Jacobi on R^T; T = P R^T Q^T, so
// the left vectors of T are the rows of R^T's permuted by P.  On the graded,
// numerically rank-deficient factors of the truncation this cuts the sweeps
// from 25-37 to 7-10 (tools: numpy model on captured configs[1] factors).
// Ab: one m x n row-major matrix; Ub (m x n, may be null: values only), Sb (n)
template <int ROWS, bool PIV>
__device__ __forceinline__ void jacobi_small_body(const double* __restrict__ Ab, int m, int n,
                                                  double* __restrict__ Ub, double* __restrict__ Sb,
                                                  int max_sweeps) {
  constexpr int JS_LD = ROWS + 2, NJ = ROWS / (2 * JS_LPP);  // NJ: double2 per lane and column
  static_assert(NJ * 2 * JS_LPP == ROWS, "rows must split over the lanes of a pair");
  extern __shared__ __align__(16) double sm_js[];
  double* W = sm_js;                       // n columns x JS_LD
  double* sig = sm_js + (size_t)n * JS_LD;  // n
  int* flag = reinterpret_cast<int*>(sig + n + (n & 1));
  int* perm = flag + 4;                    // n (PIV)
  int* lastmod = perm + n;                 // n: global round of each column's last rotation
  for (int idx = threadIdx.x; idx < n * JS_LD; idx += blockDim.x) {
    const int j = idx / JS_LD, i = idx - j * JS_LD;
    W[idx] = i < m ? Ab[(size_t)i * n + j] : 0.0;
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31, nwarps = blockDim.x >> 5;
  if constexpr (PIV) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) perm[i] = i;
    __syncthreads();
    // Partial column norms (squared) are DOWNDATED by the warp that updates
    // the column (cn[c] -= R[j][c]^2, LAPACK dgeqp3's scheme) instead of
    // being recomputed from the whole trailing block every step; a column
    // whose norm has lost half its digits since its last exact evaluation
    // (cn <= sqrt(eps) cn2) is re-evaluated by that warp on the spot.  They
    // only choose the pivot: the reflector's norm is always the exact one.
    double* cn = sig;
    double* cn2 = reinterpret_cast<double*>(lastmod + n);  // norms at the last exact evaluation
    for (int c = warp; c < n; c += nwarps) {
      const double* wc = W + c * JS_LD;
      double a = 0.0;
      for (int i = lane; i < m; i += 32) a = fma(wc[i], wc[i], a);
      a = warp_sum(a);
      if (lane == 0) cn[c] = cn2[c] = a;
    }
    __syncthreads();
    for (int j = 0; j < n; ++j) {
      if (warp == 0) {
        double best = -1.0;
        int bi = j;
        for (int c = j + lane; c < n; c += 32)
          if (cn[c] > best) {
            best = cn[c];
            bi = c;
          }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, best, o);
          const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
          if (ob > best || (ob == best && oi < bi)) {
            best = ob;
            bi = oi;
          }
        }
        if (lane == 0) flag[1] = bi;
      }
      __syncthreads();
      const int pc = flag[1];
      if (pc != j) {
        for (int i = threadIdx.x; i < m; i += blockDim.x) {
          const double t = W[j * JS_LD + i];
          W[j * JS_LD + i] = W[pc * JS_LD + i];
          W[pc * JS_LD + i] = t;
        }
        if (threadIdx.x == 0) {
          const int t = perm[j];
          perm[j] = perm[pc];
          perm[pc] = t;
          // column j's own entries are not read again
          cn[pc] = cn[j];
          cn2[pc] = cn2[j];
        }
      }
      __syncthreads();
      // Householder vector of column j (rows j..m-1): v = x - alpha e_j; its
      // norm exactly, by every warp (same data, same order: identical)
      double* wj = W + j * JS_LD;
      double xn2 = 0.0;
      for (int i = j + lane; i < m; i += 32) xn2 = fma(wj[i], wj[i], xn2);
      xn2 = warp_sum(xn2);
      const double xj = wj[j];
      const double alpha = -copysign(sqrt(xn2), xj);
      const double vj = xj - alpha;
      const double vtv = xn2 - xj * xj + vj * vj;
      if (vtv > 0.0) {
        const double beta = 2.0 / vtv;
        // four trailing columns per warp in flight (their reductions interleave)
        for (int c0 = j + 1 + warp; c0 < n; c0 += 4 * nwarps) {
          double d[4] = {0.0, 0.0, 0.0, 0.0};
          for (int i = j + lane; i < m; i += 32) {
            const double vi = i == j ? vj : wj[i];
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const int c = c0 + u * nwarps;
              d[u] = fma(vi, W[(c < n ? c : j) * JS_LD + i], d[u]);
            }
          }
#pragma unroll
          for (int o = 16; o > 0; o >>= 1) {
#pragma unroll
            for (int u = 0; u < 4; ++u) d[u] += __shfl_xor_sync(0xffffffffu, d[u], o);
          }
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int c = c0 + u * nwarps;
            if (c >= n) break;
            double* wc = W + c * JS_LD;
            const double du = d[u] * beta;
            double rjc = 0.0;
            for (int i = j + lane; i < m; i += 32) {
              const double v = fma(-du, i == j ? vj : wj[i], wc[i]);
              wc[i] = v;
              if (i == j) rjc = v;  // lane 0: R[j][c]
            }
            rjc = __shfl_sync(0xffffffffu, rjc, 0);
            const double t = cn[c] - rjc * rjc;
            if (!(t > 1.5e-8 * cn2[c])) {
              __syncwarp();
              double a = 0.0;
              for (int i = j + 1 + lane; i < m; i += 32) a = fma(wc[i], wc[i], a);
              a = warp_sum(a);
              if (lane == 0) cn[c] = cn2[c] = a;
            } else if (lane == 0) {
              cn[c] = t;
            }
          }
        }
      }
      __syncthreads();
      for (int i = j + threadIdx.x; i < m; i += blockDim.x) wj[i] = (i == j) ? (vtv > 0.0 ? alpha : xj) : 0.0;
    }
    __syncthreads();
    // W := R^T (in place; R is upper triangular)
    for (int idx = threadIdx.x; idx < n * n; idx += blockDim.x) {
      const int c = idx / n, r = idx - c * n;
      if (r < c) {
        const double t = W[c * JS_LD + r];
        W[c * JS_LD + r] = W[r * JS_LD + c];
        W[r * JS_LD + c] = t;
      }
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) lastmod[i] = -(1 << 30);
  __syncthreads();
  const int N = n + (n & 1);
  const int g = threadIdx.x / JS_LPP, l4 = threadIdx.x % JS_LPP;
  const double tol = 1e-15 * (double)m, tol2 = tol * tol;
  for (int sweep = 0; sweep < max_sweeps; ++sweep) {
    if (threadIdx.x == 0) *flag = 0;
    __syncthreads();
    for (int r = 0; r < N - 1; ++r) {
      int p, q;
      rr_pair(N, r, g, p, q);
      // every lane takes part in the reductions (full-mask shuffles); pairs
      // that do not exist read zeros and never rotate.  A pair found
      // converged one sweep ago (N - 1 rounds, the round-robin period) whose
      // columns have not been rotated since is still converged: skipped
      // without reading its columns (the late sweeps touch few pairs).
      const int gr = sweep * (N - 1) + r;
      bool live = g < N / 2 && p < n && q < n;
      if (live && sweep > 0 && lastmod[p] < gr - (N - 1) && lastmod[q] < gr - (N - 1)) live = false;
      double2* wp = reinterpret_cast<double2*>(W + (live ? p : 0) * JS_LD) + l4;
      double2* wq = reinterpret_cast<double2*>(W + (live ? q : 0) * JS_LD) + l4;
      double2 x[NJ], y[NJ];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        x[j] = live ? wp[JS_LPP * j] : make_double2(0.0, 0.0);
        y[j] = live ? wq[JS_LPP * j] : make_double2(0.0, 0.0);
      }
      double al = 0.0, be = 0.0, ga = 0.0, al2 = 0.0, be2 = 0.0, ga2 = 0.0;
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        al = fma(x[j].x, x[j].x, al);
        be = fma(y[j].x, y[j].x, be);
        ga = fma(x[j].x, y[j].x, ga);
        al2 = fma(x[j].y, x[j].y, al2);
        be2 = fma(y[j].y, y[j].y, be2);
        ga2 = fma(x[j].y, y[j].y, ga2);
      }
      al += al2;
      be += be2;
      ga += ga2;
#pragma unroll
      for (int o = JS_LPP / 2; o > 0; o >>= 1) {
        al += __shfl_xor_sync(0xffffffffu, al, o);
        be += __shfl_xor_sync(0xffffffffu, be, o);
        ga += __shfl_xor_sync(0xffffffffu, ga, o);
      }
      if (ga != 0.0 && ga * ga > tol2 * (al * be)) {
        if (l4 == 0) {
          *flag = 1;
          lastmod[p] = gr;
          lastmod[q] = gr;
        }
        const double zeta = (be - al) / (2.0 * ga);
        const double t = copysign(1.0, zeta) / (fabs(zeta) + sqrt(fma(zeta, zeta, 1.0)));
        const double c = rsqrt(fma(t, t, 1.0)), sn = c * t;
#pragma unroll
        for (int j = 0; j < NJ; ++j) {
          wp[JS_LPP * j] = make_double2(c * x[j].x - sn * y[j].x, c * x[j].y - sn * y[j].y);
          wq[JS_LPP * j] = make_double2(sn * x[j].x + c * y[j].x, sn * x[j].y + c * y[j].y);
        }
      }
      __syncthreads();
    }
    const int any = *flag;
    __syncthreads();
    if (!any) break;
  }
  // singular values = column norms, ranked by decreasing value (ties by index)
  for (int j = warp; j < n; j += nwarps) {
    const double* wj = W + j * JS_LD;
    double a = 0.0;
    for (int i = lane; i < m; i += 32) a = fma(wj[i], wj[i], a);
    a = warp_sum(a);
    if (lane == 0) sig[j] = sqrt(a);
  }
  __syncthreads();
  for (int j = warp; j < n; j += nwarps) {
    const double sj = sig[j];
    int rank = 0;
    for (int i = lane; i < n; i += 32) rank += (sig[i] > sj || (sig[i] == sj && i < j)) ? 1 : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) rank += __shfl_xor_sync(0xffffffffu, rank, o);
    if (lane == 0) Sb[rank] = sj;
    if (Ub == nullptr) continue;
    const double inv = sj > 0.0 ? 1.0 / sj : 0.0;
    const double* wj = W + j * JS_LD;
    for (int i = lane; i < m; i += 32) {
      const int row = PIV ? perm[i] : i;
      Ub[(size_t)row * n + rank] = (sj > 0.0) ? wj[i] * inv : (i == j ? 1.0 : 0.0);
    }
  }
}

template <int ROWS, bool PIV>
__global__ void __launch_bounds__(JS_THREADS, 1) k_jacobi_small(const double* __restrict__ A, int m, int n,
                                                                double* __restrict__ U, double* __restrict__ S,
                                                                int max_sweeps) {
  jacobi_small_body<ROWS, PIV>(A + (size_t)blockIdx.x * m * n, m, n, U + (size_t)blockIdx.x * m * n,
                               S + (size_t)blockIdx.x * n, max_sweeps);
}

// Pivoted small SVDs of square matrices of different sizes in one launch:
// CTA i takes the k_i x k_i matrix A_i (the R factors of tsqr_r).
struct JacobiMulti {
  const double* A[FL_QR_MAX_BATCH];
  double* U[FL_QR_MAX_BATCH];
  double* S[FL_QR_MAX_BATCH];
  int k[FL_QR_MAX_BATCH];
};

__global__ void __launch_bounds__(JS_THREADS, 1) k_jacobi_multi(const JacobiMulti jm, int max_sweeps) {
  const int i = blockIdx.x, k = jm.k[i];
  if (k <= 32)
    jacobi_small_body<32, true>(jm.A[i], k, k, jm.U[i], jm.S[i], max_sweeps);
  else if (k <= 64)
    jacobi_small_body<64, true>(jm.A[i], k, k, jm.U[i], jm.S[i], max_sweeps);
  else if (k <= 96)
    jacobi_small_body<96, true>(jm.A[i], k, k, jm.U[i], jm.S[i], max_sweeps);
  else
    jacobi_small_body<128, true>(jm.A[i], k, k, jm.U[i], jm.S[i], max_sweeps);
}

}  // namespace

constexpr size_t SVD_SMEM_CAP = 200 * 1024;
#ifndef FL_SVD_SWEEPS
#define FL_SVD_SWEEPS 40
#endif

template <int ROWS, bool PIV = false>
static int launch_jacobi_small(const double* A, int batch, int m, int n, double* U, double* S, int sweeps,
                               cudaStream_t st) {
  constexpr int LD = ROWS + 2;
  // W, sig (+1 for alignment), flag[4], perm[n], lastmod[n]
  // W, sig (+1 for alignment), flag[4], perm[n], lastmod[n], cn2[n] (PIV)
  const size_t smem = sizeof(double) * ((size_t)n * LD + 2 * (size_t)n + 2) + sizeof(int) * (4 + 2 * (size_t)n);
  const size_t smem_max = sizeof(double) * ((size_t)JS_ROWS * LD + 2 * JS_ROWS + 2) + sizeof(int) * (4 + 2 * JS_ROWS);
  static std::atomic<uint64_t> attr_js{0};
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_js.load() & bit)) {
    FL_CUDA_TRY(cudaFuncSetAttribute(k_jacobi_small<ROWS, PIV>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     (int)smem_max));
    attr_js.fetch_or(bit);
  }
  k_jacobi_small<ROWS, PIV><<<batch, JS_THREADS, smem, st>>>(A, m, n, U, S, sweeps);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// left singular system of T = A^T for square A (k x k, k <= 128) through a
// column-pivoted QR of A and Jacobi on R^T (see k_jacobi_small<.., true>)
int svd_left_pivoted(const double* A, int batch, int k, double* U, double* S, cudaStream_t st) {
  FL_ARG_CHECK(batch >= 0 && k >= 1 && k <= JS_ROWS, "pivoted small SVD: bad shape (%d, %d)", batch, k);
  if (batch == 0) return FL_OK;
  if (k <= 32) return launch_jacobi_small<32, true>(A, batch, k, k, U, S, 2 * FL_SVD_SWEEPS, st);
  if (k <= 64) return launch_jacobi_small<64, true>(A, batch, k, k, U, S, 2 * FL_SVD_SWEEPS, st);
  if (k <= 96) return launch_jacobi_small<96, true>(A, batch, k, k, U, S, 2 * FL_SVD_SWEEPS, st);
  return launch_jacobi_small<128, true>(A, batch, k, k, U, S, 2 * FL_SVD_SWEEPS, st);
}

// Left singular systems of a batch of wide matrices M_i (k_i x m_i, k_i <=
// 128): R_i of M_i^T = Q R by TSQR (qr.cu), then the pivoted Jacobi on every
// R_i in one launch.  U_i may be null (singular values only).
int left_sv_wide(int batch, const double* const* M, const int* k, const int64_t* m, const int64_t* rs,
                 const int64_t* cs, double* const* U, double* const* S, cudaStream_t st) {
  FL_ARG_CHECK(batch >= 0 && batch <= FL_QR_MAX_BATCH, "left_sv_wide: batch must be 0..%d", FL_QR_MAX_BATCH);
  if (batch == 0) return FL_OK;
  size_t total = 0, off[FL_QR_MAX_BATCH];
  int kmax = 1;
  for (int i = 0; i < batch; ++i) {
    FL_ARG_CHECK(k[i] >= 1 && k[i] <= JS_ROWS, "left_sv_wide: k = %d outside 1..%d", k[i], JS_ROWS);
    FL_ARG_CHECK(S[i] != nullptr, "left_sv_wide: null output");
    off[i] = total;
    total += (size_t)k[i] * k[i];
    if (k[i] > kmax) kmax = k[i];
  }
  DevBuf rbuf;
  int rc = rbuf.alloc((int64_t)total, st);
  if (rc) return rc;
  double* R[FL_QR_MAX_BATCH];
  for (int i = 0; i < batch; ++i) R[i] = rbuf.p + off[i];
  if ((rc = tsqr_r(batch, M, k, m, rs, cs, R, st))) return rc;
  JacobiMulti jm{};
  for (int i = 0; i < batch; ++i) {
    jm.A[i] = R[i];
    jm.U[i] = U ? U[i] : nullptr;
    jm.S[i] = S[i];
    jm.k[i] = k[i];
  }
  const int rows = kmax <= 32 ? 32 : kmax <= 64 ? 64 : kmax <= 96 ? 96 : 128;
  const size_t smem = sizeof(double) * ((size_t)kmax * (rows + 2) + 2 * (size_t)kmax + 2) + sizeof(int) * (4 + 2 * (size_t)kmax);
  const size_t smem_max = sizeof(double) * ((size_t)JS_ROWS * (JS_ROWS + 2) + 2 * JS_ROWS + 2) + sizeof(int) * (4 + 2 * JS_ROWS);
  static std::atomic<uint64_t> attr_jm{0};
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_jm.load() & bit)) {
    FL_CUDA_TRY(cudaFuncSetAttribute(k_jacobi_multi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem_max));
    attr_jm.fetch_or(bit);
  }
  k_jacobi_multi<<<batch, JS_THREADS, smem, st>>>(jm, 2 * FL_SVD_SWEEPS);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

static bool small_svd_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FL_SMALL_SVD");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

int svd_batched(const double* A, int batch, int m, int n, double* U, double* S, double* Vt, cudaStream_t st) {
  FL_ARG_CHECK(batch >= 0 && m >= 1 && n >= 1, "bad batched SVD shape (%d, %d, %d)", batch, m, n);
  FL_ARG_CHECK(Vt != nullptr || m >= n, "batched SVD without Vt needs m >= n, got %d x %d", m, n);
  const size_t M = m > n ? m : n, K = m < n ? m : n;
  const size_t wb = sizeof(double) * M * K, vb = Vt ? sizeof(double) * K * K : 0, tail = sizeof(double) * K + 2 * sizeof(int);
  FL_ARG_CHECK(tail <= SVD_SMEM_CAP, "batched SVD: %d x %d matrices are too large", m, n);
  if (batch == 0) return FL_OK;
#ifndef FL_SVD_SWEEPS
#define FL_SVD_SWEEPS 40
#endif
  if (Vt == nullptr && m <= JS_ROWS && n <= JS_ROWS && small_svd_enabled()) {
    // graded, numerically rank-deficient factors need more sweeps than random
    // matrices (~30 measured on configs[1] factors)
    if (m <= 32) return launch_jacobi_small<32>(A, batch, m, n, U, S, 2 * FL_SVD_SWEEPS, st);
    if (m <= 64) return launch_jacobi_small<64>(A, batch, m, n, U, S, 2 * FL_SVD_SWEEPS, st);
    if (m <= 96) return launch_jacobi_small<96>(A, batch, m, n, U, S, 2 * FL_SVD_SWEEPS, st);
    return launch_jacobi_small<128>(A, batch, m, n, U, S, 2 * FL_SVD_SWEEPS, st);
  }
  int w_sm = 0, v_sm = 0;
  if (wb + vb + tail <= SVD_SMEM_CAP) {
    w_sm = v_sm = 1;
  } else if (wb + tail <= SVD_SMEM_CAP) {
    w_sm = 1;
  }
  const size_t smem = (w_sm ? wb : 0) + (v_sm ? vb : 0) + tail;
  double* scratch = nullptr;
  // per-matrix scratch stride, the same one the kernel indexes with
  const size_t gstride = M * K + (Vt ? K * K : 0);
  if (!(w_sm && v_sm)) {
    if (int rc = keep_pool_cached()) return rc;
  }
  if (!(w_sm && v_sm)) FL_CUDA_TRY(cudaMallocAsync(&scratch, sizeof(double) * gstride * (size_t)batch, st));
  // function attributes are per device: one flag bit per device ordinal
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load() & bit)) {
    FL_CUDA_TRY(cudaFuncSetAttribute(k_svd_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SVD_SMEM_CAP));
    attr_set.fetch_or(bit);
  }
  k_svd_jacobi<<<batch, SVD_THREADS, smem, st>>>(A, m, n, U, S, Vt, FL_SVD_SWEEPS, scratch, gstride, w_sm, v_sm);
  FL_LAUNCH_CHECK();
  if (scratch) FL_CUDA_TRY(cudaFreeAsync(scratch, st));
  return FL_OK;
}

}  // namespace fl
