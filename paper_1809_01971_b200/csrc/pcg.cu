// Full-format preconditioned CG in spectral space.
//
// The operator F diag(A) F and the preconditioner F diag(P) F share the
// orthonormal per-mode DST-I basis F, so PCG (reference solver.py:116-180)
// runs on the spectral coefficients with diagonal scalings only; inner
// products are preserved by Parseval.  The iteration is identical to the
// nodal one up to rounding, with one forward transform of b and one inverse
// transform of x for the whole solve.
//
// One streaming pass per iteration (64 B/DoF: read p, r, x, A, P; write p,
// x, r).  Pass j forms the search direction of the reference's iteration on
// the fly, p_j = P r_j + beta_j p_{j-1}, applies the update x += alpha_j p_j,
// r -= alpha_j A p_j, and accumulates the four sums the next iteration needs
// with z = P r_{j+1}:
//   rr = <r, r> (stopping rule), rz = <r, z>, eta = <z, A z>, mu = <z, A p_j>.
// Then beta_{j+1} = rz_{j+1} / rz_j and, exactly (p_{j+1} = z + beta p_j),
//   <p_{j+1}, A p_{j+1}> = eta + 2 beta mu + beta^2 <p_j, A p_j>,
// so x, r and p are the reference iteration's vectors; only <P,S> is formed
// from the expansion instead of a second pass (the earlier two-phase kernel
// streamed 96 B/DoF per iteration).  The breakdown tests (<R,Z> <= 0, then
// <P,S> <= 0) are evaluated in the reference's order.
//
// k_pcg_spectral: one cooperative persistent launch for the whole solve, one
// grid barrier per iteration (block partials double-buffered by iteration
// parity, re-summed in the same order by every block, so every block takes
// the same decisions).  No host round trip per iteration.
//
// Phase kernels (k_pcg_init / k_pcg_step): the same passes as separate
// launches whose partial sums are reduced across GPUs by the caller (NCCL),
// for the slab-partitioned multi-GPU solve: one all-reduce of 4 scalars per
// iteration.
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace fl {

constexpr int PCG_NT = 512;

struct PcgArgs {
  const double* b;  // spectral right-hand side
  double* x;
  double* r;
  double* p;
  const double* A;
  const double* P;
  int64_t N;
  double tol;
  int kmax;
  double* hist;        // kmax + 1 relative residuals (breakdown: the offending value at its iteration)
  int* status;         // [iterations, converged, breakdown iteration, breakdown kind (1: <R,Z>, 2: <P,S>)]
  double* partial;     // 2 * gridDim.x * 4 block partials (double-buffered)
  unsigned* bar;       // [count, generation]
};

__device__ __forceinline__ double block_sum(double v, double* sh) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) sh[w] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x < 32) {
    t = (threadIdx.x < (blockDim.x >> 5)) ? sh[threadIdx.x] : 0.0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  }
  return t;  // valid in thread 0
}

__device__ __forceinline__ void grid_barrier(unsigned* bar, unsigned nblocks) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* gen = bar + 1;
    const unsigned g = *gen;
    __threadfence();
    if (atomicAdd(bar, 1u) == nblocks - 1) {
      bar[0] = 0;
      __threadfence();
      atomicAdd(bar + 1, 1u);
    } else {
      while (*gen == g) {
      }
    }
    __threadfence();
  }
  __syncthreads();
}

// sums of the 4 block partials of set `set`, same order in every block;
// returned in every thread
__device__ __forceinline__ void all_partials4(const double* partial, int nb, double* sh, double (&out)[4]) {
  __shared__ double bc[4];
  for (int k = 0; k < 4; ++k) {
    double v = 0.0;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) v += partial[4 * i + k];
    const double t = block_sum(v, sh);
    if (threadIdx.x == 0) bc[k] = t;
  }
  __syncthreads();
#pragma unroll
  for (int k = 0; k < 4; ++k) out[k] = bc[k];
  __syncthreads();
}

__device__ __forceinline__ void put_partials4(double* partial, double v0, double v1, double v2, double v3,
                                              double* sh) {
  v0 = block_sum(v0, sh);
  v1 = block_sum(v1, sh);
  v2 = block_sum(v2, sh);
  v3 = block_sum(v3, sh);
  if (threadIdx.x == 0) {
    partial[4 * blockIdx.x + 0] = v0;
    partial[4 * blockIdx.x + 1] = v1;
    partial[4 * blockIdx.x + 2] = v2;
    partial[4 * blockIdx.x + 3] = v3;
  }
}

// one streaming pass (see the header): p = P r + beta p; x += alpha p;
// r -= alpha A p; sums of r.r, r.Pr, (Pr).A(Pr), (Pr).A p over this thread's
// elements
__device__ __forceinline__ void pcg_pass(double* __restrict__ x, double* __restrict__ r, double* __restrict__ p,
                                         const double* __restrict__ A, const double* __restrict__ P, int64_t i0,
                                         int64_t stride, int64_t N, double alpha, double beta, double& rr,
                                         double& rz, double& eta, double& mu) {
  for (int64_t i = i0; i < N; i += stride) {
    const double ai = A[i], qi = P[i];
    const double pi = fma(beta, p[i], qi * r[i]);
    const double ri = fma(-alpha, ai * pi, r[i]);
    x[i] = fma(alpha, pi, x[i]);
    r[i] = ri;
    p[i] = pi;
    const double zi = qi * ri, azi = ai * zi;
    rr = fma(ri, ri, rr);
    rz = fma(ri, zi, rz);
    eta = fma(azi, zi, eta);
    mu = fma(azi, pi, mu);
  }
}

__global__ void __launch_bounds__(PCG_NT) k_pcg_spectral(const PcgArgs a) {
  __shared__ double sh[PCG_NT / 32];
  const int nb = gridDim.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // init: x = 0, r = b, p = 0 (p_{-1}); sums b.b, <b, P b>, <P b, A P b>
  double bb = 0.0, rz = 0.0, eta = 0.0;
  for (int64_t i = i0; i < a.N; i += stride) {
    const double bi = a.b[i];
    const double zi = a.P[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.p[i] = 0.0;
    bb = fma(bi, bi, bb);
    rz = fma(bi, zi, rz);
    eta = fma(zi * a.A[i], zi, eta);
  }
  put_partials4(a.partial, bb, rz, eta, 0.0, sh);
  grid_barrier(a.bar, nb);
  double s4[4];
  all_partials4(a.partial, nb, sh, s4);
  const double norm_b = sqrt(s4[0]);
  rz = s4[1];
  double ps = s4[2], beta = 0.0;  // p_0 = z_0: <p_0, A p_0> = eta_0
  if (norm_b == 0.0) {
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      a.hist[0] = 0.0;
      a.status[0] = 0;
      a.status[1] = 1;
    }
    return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[0] = 1.0;
  int k = 1;
  int converged = 0, bk_iter = 0, bk_kind = 0;
  for (; k <= a.kmax; ++k) {
    if (!(rz > 0.0)) {
      bk_iter = k;
      bk_kind = 1;
      break;
    }
    if (!(ps > 0.0)) {
      bk_iter = k;
      bk_kind = 2;
      break;
    }
    const double alpha = rz / ps;
    double rr = 0.0, rzn = 0.0, etan = 0.0, mu = 0.0;
    pcg_pass(a.x, a.r, a.p, a.A, a.P, i0, stride, a.N, alpha, beta, rr, rzn, etan, mu);
    double* part = a.partial + (size_t)(k & 1) * 4 * nb;
    put_partials4(part, rr, rzn, etan, mu, sh);
    grid_barrier(a.bar, nb);
    all_partials4(part, nb, sh, s4);
    const double rel = sqrt(fmax(s4[0], 0.0)) / norm_b;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = rel;
    if (rel <= a.tol) {
      converged = 1;
      break;
    }
    // next direction p_{k+1} = z + beta p_k: its A-norm from the expansion
    const double bn = s4[1] / rz;
    ps = s4[2] + 2.0 * bn * s4[3] + bn * bn * ps;
    beta = bn;
    rz = s4[1];
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    // on breakdown the slot of the failed iteration carries the nonpositive
    // <R,Z> or <P,S> (the value the reference reports, solver.py:154-159)
    if (bk_kind) a.hist[bk_iter] = (bk_kind == 1) ? rz : ps;
    a.status[0] = converged ? k : (bk_kind ? bk_iter - 1 : a.kmax);
    a.status[1] = converged;
    a.status[2] = bk_iter;
    a.status[3] = bk_kind;
  }
}

int pcg_spectral(const double* b, double* x, double* r, double* p, const double* A, const double* P, int64_t N,
                 double tol, int kmax, double* hist, int* status, cudaStream_t st) {
  FL_ARG_CHECK(N >= 1 && kmax >= 1, "bad PCG arguments");
  static int occ = 0;
  if (occ == 0) {
    FL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_pcg_spectral, PCG_NT, 0));
    if (occ < 1) occ = 1;
  }
  int64_t want = (N + PCG_NT - 1) / PCG_NT;
  int64_t cap = (int64_t)occ * sm_count();
  const int grid = (int)(want < cap ? (want < 1 ? 1 : want) : cap);
  DevBuf partial, bar;
  int rc;
  if ((rc = partial.alloc((int64_t)8 * grid, st))) return rc;
  if ((rc = bar.alloc(1, st))) return rc;
  unsigned* barp = reinterpret_cast<unsigned*>(bar.p);
  FL_CUDA_TRY(cudaMemsetAsync(barp, 0, sizeof(unsigned) * 2, st));
  PcgArgs a{b, x, r, p, A, P, N, tol, kmax, hist, status, partial.p, barp};
  void* args[] = {&a};
  FL_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_pcg_spectral, dim3(grid), dim3(PCG_NT), args, 0, st));
  return FL_OK;
}

// ---------------------------------------------------------------------------
// phase kernels (multi-GPU): local partial sums land in out[] via a
// deterministic last-block reduction
// ---------------------------------------------------------------------------
struct PhaseArgs {
  const double* b;
  double* x;
  double* r;
  double* p;
  const double* A;
  const double* P;
  int64_t N;
  double alpha, beta;  // step: update step and direction coefficient
  double* part;        // gridDim.x * 4
  double* out;         // 4 sums
  unsigned* done;
};

__device__ __forceinline__ void finish_sums4(const PhaseArgs& a, double v0, double v1, double v2, double v3,
                                             double* sh) {
  put_partials4(a.part, v0, v1, v2, v3, sh);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    __threadfence();
    last = (atomicAdd(a.done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    __threadfence();
    for (int k = 0; k < 4; ++k) {
      double v = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += a.part[4 * i + k];
      v = block_sum(v, sh);
      if (threadIdx.x == 0) a.out[k] = v;
    }
    if (threadIdx.x == 0) *a.done = 0;
  }
}

// x = 0, r = b, p = 0; out = [b.b, <b, P b>, <P b, A P b>, 0]
__global__ void __launch_bounds__(PCG_NT) k_pcg_init(const PhaseArgs a) {
  __shared__ double sh[PCG_NT / 32];
  double bb = 0.0, rz = 0.0, eta = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.N; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = a.b[i];
    const double zi = a.P[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.p[i] = 0.0;
    bb = fma(bi, bi, bb);
    rz = fma(bi, zi, rz);
    eta = fma(zi * a.A[i], zi, eta);
  }
  finish_sums4(a, bb, rz, eta, 0.0, sh);
}

// the single pass of k_pcg_spectral; out = [r.r, r.Pr, (Pr).A(Pr), (Pr).A p]
__global__ void __launch_bounds__(PCG_NT) k_pcg_step(const PhaseArgs a) {
  __shared__ double sh[PCG_NT / 32];
  double rr = 0.0, rz = 0.0, eta = 0.0, mu = 0.0;
  pcg_pass(a.x, a.r, a.p, a.A, a.P, (int64_t)blockIdx.x * blockDim.x + threadIdx.x,
           (int64_t)gridDim.x * blockDim.x, a.N, a.alpha, a.beta, rr, rz, eta, mu);
  finish_sums4(a, rr, rz, eta, mu, sh);
}

int pcg_phase(int which, const double* b, double* x, double* r, double* p, const double* A, const double* P,
              int64_t N, double alpha, double beta, double* out, double* work, cudaStream_t st) {
  FL_ARG_CHECK(which == 0 || which == 1, "unknown PCG phase %d", which);
  int grid = sm_count() * 2;
  const int64_t want = (N + PCG_NT - 1) / PCG_NT;
  if (want < grid) grid = (int)(want < 1 ? 1 : want);
  // work: FL_PCG_WORK doubles, zero-initialised once by the caller; block
  // partials at the front, the completion counter in the last slot
  PhaseArgs a{b, x, r, p, A, P, N, alpha, beta, work, out, reinterpret_cast<unsigned*>(work + FL_PCG_WORK - 1)};
  if (which == 0) k_pcg_init<<<grid, PCG_NT, 0, st>>>(a);
  if (which == 1) k_pcg_step<<<grid, PCG_NT, 0, st>>>(a);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

}  // namespace fl
