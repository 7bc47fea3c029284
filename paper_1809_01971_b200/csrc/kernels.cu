// Dense fp64 building blocks: core evaluation, CP expansion, sinc factors
// and small elementwise kernels (the DMMA GEMM is in gemm_dmma.cu).
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace fl {

// ---------------------------------------------------------------------------
// elementwise
// ---------------------------------------------------------------------------
__global__ void k_ew_mul(const double* __restrict__ a, const double* __restrict__ b, double* out, int64_t count,
                         double scale) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = scale * a[i] * b[i];
}

static int ew_grid(int64_t count) {
  int64_t g = (count + 255) / 256;
  const int64_t cap = (int64_t)sm_count() * 8;
  if (g > cap) g = cap;
  return (int)(g < 1 ? 1 : g);
}

int ew_mul(const double* a, const double* b, double* out, int64_t count, double scale, cudaStream_t st) {
  if (count <= 0) return FL_OK;
  k_ew_mul<<<ew_grid(count), 256, 0, st>>>(a, b, out, count, scale);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

__global__ void k_kr_expand(const double* __restrict__ U, const double* __restrict__ Xs, double* out, int64_t n,
                            int64_t R, int64_t S) {
  const int64_t total = n * R * S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / (R * S), c = i % (R * S);
    const int64_t k = c / S, s = c % S;
    out[i] = U[j * R + k] * Xs[j * S + s];
  }
}

int kr_expand(const double* U, const double* Xs, double* out, int64_t n, int64_t R, int64_t S, cudaStream_t st) {
  const int64_t total = n * R * S;
  if (total <= 0) return FL_OK;
  k_kr_expand<<<ew_grid(total), 256, 0, st>>>(U, Xs, out, n, R, S);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// ---------------------------------------------------------------------------
// cores
// ---------------------------------------------------------------------------
struct CoreArgs {
  int d;
  int64_t n0, n1, n2;
  const double* mu0;
  const double* mu1;
  const double* mu2;
  int tag;
  double a, cm, cp;
  int recip;
};

// fracop.py:109-121 _eval_on_rho
__device__ __forceinline__ double eval_on_rho(const CoreArgs& c, double rho) {
  if (c.tag == FL_G1) {
    const double v = c.cm * pow(rho, -c.a);
    return c.recip ? 1.0 / v : v;
  }
  if (c.tag == FL_G2 || c.tag == FL_G3) {
    const double s = c.cm * pow(rho, -c.a) + c.cp * pow(rho, c.a);
    const bool want_sum = (c.tag == FL_G2) != (c.recip != 0);
    return want_sum ? s : 1.0 / s;
  }
  const double s = 1.0 + c.cp * pow(rho, 2.0 * c.a);
  return c.recip ? s : 1.0 / s;
}

__global__ void k_core_eval(double* out, const CoreArgs c) {
  const int64_t total = c.n0 * c.n1 * (c.d == 3 ? c.n2 : 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double rho;
    if (c.d == 2) {
      const int64_t i0 = i / c.n1, i1 = i % c.n1;
      rho = c.mu0[i0] + c.mu1[i1];
    } else {
      const int64_t i2 = i % c.n2, r = i / c.n2;
      const int64_t i1 = r % c.n1, i0 = r / c.n1;
      rho = (c.mu0[i0] + c.mu1[i1]) + c.mu2[i2];
    }
    out[i] = eval_on_rho(c, rho);
  }
}

struct CpDenseArgs {
  int d;
  int64_t n0, n1, n2, R;
  const double* w;
  const double* U0;
  const double* U1;
  const double* U2;
};

__global__ void k_cp_to_dense(double* out, const CpDenseArgs c) {
  const int64_t total = c.n0 * c.n1 * (c.d == 3 ? c.n2 : 1);
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    double acc = 0.0;
    if (c.d == 2) {
      const int64_t i0 = i / c.n1, i1 = i % c.n1;
      const double* u0 = c.U0 + i0 * c.R;
      const double* u1 = c.U1 + i1 * c.R;
      for (int64_t k = 0; k < c.R; ++k) acc = fma(c.w[k] * u0[k], u1[k], acc);
    } else {
      const int64_t i2 = i % c.n2, r = i / c.n2;
      const int64_t i1 = r % c.n1, i0 = r / c.n1;
      const double* u0 = c.U0 + i0 * c.R;
      const double* u1 = c.U1 + i1 * c.R;
      const double* u2 = c.U2 + i2 * c.R;
      for (int64_t k = 0; k < c.R; ++k) acc = fma(c.w[k] * u0[k] * u1[k], u2[k], acc);
    }
    out[i] = acc;
  }
}

__global__ void k_sinc_factor(double* U, const double* __restrict__ mu, int64_t n, const double* __restrict__ t,
                              int64_t R, double rho_min) {
  const int64_t total = n * R;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t j = i / R, k = i % R;
    U[i] = exp(-((mu[j] / rho_min) * t[k]));
  }
}

int core_eval(double* out, int d, const int64_t* dims, const double* const* mu, int tag, double a, double cm,
              double cp, int recip, cudaStream_t st) {
  FL_ARG_CHECK(d == 2 || d == 3, "only tensors of order 2 or 3 are supported");
  FL_ARG_CHECK(tag >= FL_G1 && tag <= FL_G4, "unknown core function tag %d", tag);
  CoreArgs c{d, dims[0], dims[1], d == 3 ? dims[2] : 1, mu[0], mu[1], d == 3 ? mu[2] : nullptr, tag, a, cm, cp,
             recip};
  const int64_t total = c.n0 * c.n1 * c.n2;
  if (total <= 0) return FL_OK;
  k_core_eval<<<ew_grid(total), 256, 0, st>>>(out, c);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int cp_to_dense(double* out, int d, const int64_t* dims, int64_t R, const double* w, const double* const* U,
                cudaStream_t st) {
  FL_ARG_CHECK(d == 2 || d == 3, "only tensors of order 2 or 3 are supported");
  const int64_t total = dims[0] * dims[1] * (d == 3 ? dims[2] : 1);
  if (total <= 0) return FL_OK;
  if (R == 0) {
    FL_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * total, st));
    return FL_OK;
  }
  CpDenseArgs c{d, dims[0], dims[1], d == 3 ? dims[2] : 1, R, w, U[0], U[1], d == 3 ? U[2] : nullptr};
  k_cp_to_dense<<<ew_grid(total), 256, 0, st>>>(out, c);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int sinc_factor(double* U, const double* mu, int64_t n, const double* t, int64_t R, double rho_min,
                cudaStream_t st) {
  if (n * R <= 0) return FL_OK;
  k_sinc_factor<<<ew_grid(n * R), 256, 0, st>>>(U, mu, n, t, R, rho_min);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

}  // namespace fl
