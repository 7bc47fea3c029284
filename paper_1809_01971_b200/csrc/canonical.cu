// Canonical-format kernels: Hadamard product of per-mode Gram matrices
// (cp_inner, tensor.py:156-167; merge/ALS Gram products, decomp.py:559-589),
// column norms (cp_normalize, tensor.py:180-197), weighted inner products.
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

struct GramArgs {
  int d;
  int64_t n[3];
  const double* A[3];
  const double* B[3];
  int64_t Ra, Rb;
  double* H;  // Ra x Rb, row-major
};

// H[i][j] = prod_l sum_r A_l[r][i] * B_l[r][j]; 32x32 output tile per CTA,
// 256 threads (each 4 outputs), rows of the factor matrices staged in smem.
__global__ void __launch_bounds__(256) k_gram_hadamard(const GramArgs g) {
  constexpr int T = 32, KR = 32;
  __shared__ double As[KR][T + 1];
  __shared__ double Bs[KR][T + 1];
  const int64_t i0 = (int64_t)blockIdx.y * T, j0 = (int64_t)blockIdx.x * T;
  const int tx = threadIdx.x % 32, ty = threadIdx.x / 32;  // ty in [0, 8)
  double prod[4] = {1.0, 1.0, 1.0, 1.0};
  for (int l = 0; l < g.d; ++l) {
    const double* A = g.A[l];
    const double* B = g.B[l];
    const int64_t n = g.n[l];
    double acc[4] = {0.0, 0.0, 0.0, 0.0};
    for (int64_t r0 = 0; r0 < n; r0 += KR) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int rr = ty + 8 * q;
        const int64_t r = r0 + rr;
        As[rr][tx] = (r < n && i0 + tx < g.Ra) ? A[r * g.Ra + i0 + tx] : 0.0;
        Bs[rr][tx] = (r < n && j0 + tx < g.Rb) ? B[r * g.Rb + j0 + tx] : 0.0;
      }
      __syncthreads();
#pragma unroll 8
      for (int rr = 0; rr < KR; ++rr) {
        const double b = Bs[rr][tx];
#pragma unroll
        for (int q = 0; q < 4; ++q) acc[q] = fma(As[rr][ty + 8 * q], b, acc[q]);
      }
      __syncthreads();
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) prod[q] *= acc[q];
  }
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int64_t i = i0 + ty + 8 * q, j = j0 + tx;
    if (i < g.Ra && j < g.Rb) g.H[i * g.Rb + j] = prod[q];
  }
}

int gram_hadamard(int d, const int64_t* n, const double* const* A, int64_t Ra, const double* const* B, int64_t Rb,
                  double* H, cudaStream_t st) {
  FL_ARG_CHECK(d >= 1 && d <= 3, "order must be 1..3");
  if (Ra <= 0 || Rb <= 0) return FL_OK;
  GramArgs g{};
  g.d = d;
  for (int l = 0; l < d; ++l) {
    g.n[l] = n[l];
    g.A[l] = A[l];
    g.B[l] = B[l];
  }
  g.Ra = Ra;
  g.Rb = Rb;
  g.H = H;
  dim3 grid((unsigned)((Rb + 31) / 32), (unsigned)((Ra + 31) / 32));
  k_gram_hadamard<<<grid, 256, 0, st>>>(g);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// column norms of an (n, R) row-major matrix: one warp per column block
__global__ void k_col_norms(const double* __restrict__ U, int64_t n, int64_t R, double* out) {
  const int64_t c = (int64_t)blockIdx.x * 32 + (threadIdx.x % 32);
  const int w = threadIdx.x / 32;  // 8 warps split the rows
  __shared__ double part[8][33];
  double s = 0.0;
  if (c < R)
    for (int64_t r = w; r < n; r += 8) {
      const double v = U[r * R + c];
      s = fma(v, v, s);
    }
  part[w][threadIdx.x % 32] = s;
  __syncthreads();
  if (w == 0 && c < R) {
    double t = 0.0;
#pragma unroll
    for (int q = 0; q < 8; ++q) t += part[q][threadIdx.x];
    out[c] = sqrt(t);
  }
}

int col_norms(const double* U, int64_t n, int64_t R, double* out, cudaStream_t st) {
  if (R <= 0) return FL_OK;
  k_col_norms<<<(unsigned)((R + 31) / 32), 256, 0, st>>>(U, n, R, out);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// out[c] scaled columns: V[r][c] = U[r][c] / nrm[c] (nrm == 0 -> e_1 column)
// V may alias U (in-place normalisation): every element is read and written
// by the same thread.  Threads run along the columns (R fastest, coalesced),
// blocks stride over the rows: no 64-bit division per element; the divide
// (not a reciprocal multiply) keeps the reference's rounding of U / nrm.
__global__ void k_col_scale(const double* U, const double* __restrict__ nrm, int64_t n, int64_t R, double* V) {
  for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < R; c += (int64_t)gridDim.x * blockDim.x) {
    const double s = nrm[c];
    for (int64_t r = blockIdx.y; r < n; r += gridDim.y) {
      const int64_t i = r * R + c;
      V[i] = (s == 0.0) ? (r == 0 ? 1.0 : 0.0) : U[i] / s;
    }
  }
}

int col_scale(const double* U, const double* nrm, int64_t n, int64_t R, double* V, cudaStream_t st) {
  if (n * R <= 0) return FL_OK;
  int64_t gx = (R + 255) / 256;
  if (gx > 65535) gx = 65535;
  int64_t gy = ((int64_t)sm_count() * 8 + gx - 1) / gx;
  if (gy > n) gy = n;
  if (gy > 65535) gy = 65535;
  if (gy < 1) gy = 1;
  k_col_scale<<<dim3((unsigned)gx, (unsigned)gy), 256, 0, st>>>(U, nrm, n, R, V);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

}  // namespace fl
