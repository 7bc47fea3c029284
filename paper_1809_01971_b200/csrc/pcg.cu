// Full-format preconditioned CG in spectral space.
//
// The operator F diag(A) F and the preconditioner F diag(P) F share the
// orthonormal per-mode DST-I basis F, so PCG (reference solver.py:116-180)
// runs on the spectral coefficients with diagonal scalings only; inner
// products are preserved by Parseval.  The iteration is identical to the
// nodal one up to rounding, with one forward transform of b and one inverse
// transform of x for the whole solve.
//
// k_pcg_spectral: one cooperative persistent launch for the whole solve:
// grid-stride streaming phases separated by a grid barrier, deterministic
// block-partial reductions re-summed in the same order by every block, the
// stopping rule evaluated redundantly (uniformly) by all blocks.  No host
// round trip per iteration.
//
// Phase kernels (k_pcg_*): the same three streaming phases as separate
// launches whose partial sums are reduced across GPUs by the caller (NCCL),
// for the slab-partitioned multi-GPU solve.
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
  double* partial;     // gridDim.x * 3 block partials
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

// sum of the k-th partial over all blocks, same order in every block
__device__ __forceinline__ double all_partials(const double* partial, int k, int nb, double* sh) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) v += partial[3 * i + k];
  const double t = block_sum(v, sh);
  __shared__ double bc;
  if (threadIdx.x == 0) bc = t;
  __syncthreads();
  const double out = bc;
  __syncthreads();
  return out;
}

__global__ void __launch_bounds__(PCG_NT) k_pcg_spectral(const PcgArgs a) {
  __shared__ double sh[PCG_NT / 32];
  const int nb = gridDim.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  const int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // init: x = 0, r = b, p = P b; partials: bb, rz, ps
  double bb = 0.0, rz = 0.0, ps = 0.0;
  for (int64_t i = i0; i < a.N; i += stride) {
    const double bi = a.b[i];
    const double zi = a.P[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.p[i] = zi;
    bb = fma(bi, bi, bb);
    rz = fma(bi, zi, rz);
    ps = fma(zi * a.A[i], zi, ps);
  }
  bb = block_sum(bb, sh);
  rz = block_sum(rz, sh);
  ps = block_sum(ps, sh);
  if (threadIdx.x == 0) {
    a.partial[3 * blockIdx.x + 0] = bb;
    a.partial[3 * blockIdx.x + 1] = rz;
    a.partial[3 * blockIdx.x + 2] = ps;
  }
  grid_barrier(a.bar, nb);
  const double norm_b = sqrt(all_partials(a.partial, 0, nb, sh));
  rz = all_partials(a.partial, 1, nb, sh);
  ps = all_partials(a.partial, 2, nb, sh);
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
    grid_barrier(a.bar, nb);  // everyone has read the previous partials
    const double step = rz / ps;
    double rr = 0.0, rzn = 0.0;
    for (int64_t i = i0; i < a.N; i += stride) {
      const double pi = a.p[i];
      const double ri = fma(-step, a.A[i] * pi, a.r[i]);
      a.x[i] = fma(step, pi, a.x[i]);
      a.r[i] = ri;
      rr = fma(ri, ri, rr);
      rzn = fma(ri * a.P[i], ri, rzn);
    }
    rr = block_sum(rr, sh);
    rzn = block_sum(rzn, sh);
    if (threadIdx.x == 0) {
      a.partial[3 * blockIdx.x + 0] = rr;
      a.partial[3 * blockIdx.x + 1] = rzn;
    }
    grid_barrier(a.bar, nb);
    const double rel = sqrt(fmax(all_partials(a.partial, 0, nb, sh), 0.0)) / norm_b;
    rzn = all_partials(a.partial, 1, nb, sh);
    if (blockIdx.x == 0 && threadIdx.x == 0) a.hist[k] = rel;
    if (rel <= a.tol) {
      converged = 1;
      break;
    }
    grid_barrier(a.bar, nb);
    const double beta = rzn / rz;
    double psn = 0.0;
    for (int64_t i = i0; i < a.N; i += stride) {
      const double pi = fma(beta, a.p[i], a.P[i] * a.r[i]);
      a.p[i] = pi;
      psn = fma(pi * a.A[i], pi, psn);
    }
    psn = block_sum(psn, sh);
    if (threadIdx.x == 0) a.partial[3 * blockIdx.x + 2] = psn;
    grid_barrier(a.bar, nb);
    ps = all_partials(a.partial, 2, nb, sh);
    rz = rzn;
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
  double* partial = nullptr;
  unsigned* bar = nullptr;
  FL_CUDA_TRY(cudaMallocAsync(&partial, sizeof(double) * 3 * grid, st));
  FL_CUDA_TRY(cudaMallocAsync(&bar, sizeof(unsigned) * 2, st));
  FL_CUDA_TRY(cudaMemsetAsync(bar, 0, sizeof(unsigned) * 2, st));
  PcgArgs a{b, x, r, p, A, P, N, tol, kmax, hist, status, partial, bar};
  void* args[] = {&a};
  FL_CUDA_TRY(cudaLaunchCooperativeKernel((void*)k_pcg_spectral, dim3(grid), dim3(PCG_NT), args, 0, st));
  FL_CUDA_TRY(cudaFreeAsync(partial, st));
  FL_CUDA_TRY(cudaFreeAsync(bar, st));
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
  double s;      // step (update) or beta (direction)
  double* part;  // gridDim.x * 3
  double* out;   // 3 sums
  unsigned* done;
};

__device__ __forceinline__ void finish_sums(const PhaseArgs& a, double v0, double v1, double v2, int nsum, double* sh) {
  v0 = block_sum(v0, sh);
  if (nsum > 1) v1 = block_sum(v1, sh);
  if (nsum > 2) v2 = block_sum(v2, sh);
  __shared__ bool last;
  if (threadIdx.x == 0) {
    a.part[3 * blockIdx.x + 0] = v0;
    a.part[3 * blockIdx.x + 1] = v1;
    a.part[3 * blockIdx.x + 2] = v2;
    __threadfence();
    last = (atomicAdd(a.done, 1u) == gridDim.x - 1);
  }
  __syncthreads();
  if (last) {
    for (int k = 0; k < nsum; ++k) {
      double v = 0.0;
      for (int i = threadIdx.x; i < (int)gridDim.x; i += blockDim.x) v += a.part[3 * i + k];
      v = block_sum(v, sh);
      if (threadIdx.x == 0) a.out[k] = v;
    }
    if (threadIdx.x == 0) *a.done = 0;
  }
}

// r = b, p = P b, x = 0; out = [b.b, b.Pb, p.Ap]
__global__ void __launch_bounds__(PCG_NT) k_pcg_init(const PhaseArgs a) {
  __shared__ double sh[PCG_NT / 32];
  double bb = 0.0, rz = 0.0, ps = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.N; i += (int64_t)gridDim.x * blockDim.x) {
    const double bi = a.b[i];
    const double zi = a.P[i] * bi;
    a.x[i] = 0.0;
    a.r[i] = bi;
    a.p[i] = zi;
    bb = fma(bi, bi, bb);
    rz = fma(bi, zi, rz);
    ps = fma(zi * a.A[i], zi, ps);
  }
  finish_sums(a, bb, rz, ps, 3, sh);
}

// x += s p, r -= s A p; out = [r.r, r.Pr]
__global__ void __launch_bounds__(PCG_NT) k_pcg_update(const PhaseArgs a) {
  __shared__ double sh[PCG_NT / 32];
  double rr = 0.0, rz = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.N; i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = a.p[i];
    const double ri = fma(-a.s, a.A[i] * pi, a.r[i]);
    a.x[i] = fma(a.s, pi, a.x[i]);
    a.r[i] = ri;
    rr = fma(ri, ri, rr);
    rz = fma(ri * a.P[i], ri, rz);
  }
  finish_sums(a, rr, rz, 0.0, 2, sh);
}

// p = P r + s p; out = [p.Ap]
__global__ void __launch_bounds__(PCG_NT) k_pcg_direction(const PhaseArgs a) {
  __shared__ double sh[PCG_NT / 32];
  double ps = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < a.N; i += (int64_t)gridDim.x * blockDim.x) {
    const double pi = fma(a.s, a.p[i], a.P[i] * a.r[i]);
    a.p[i] = pi;
    ps = fma(pi * a.A[i], pi, ps);
  }
  finish_sums(a, ps, 0.0, 0.0, 1, sh);
}

int pcg_phase(int which, const double* b, double* x, double* r, double* p, const double* A, const double* P,
              int64_t N, double s, double* out, double* work, cudaStream_t st) {
  FL_ARG_CHECK(which >= 0 && which <= 2, "unknown PCG phase %d", which);
  int grid = sm_count() * 2;
  const int64_t want = (N + PCG_NT - 1) / PCG_NT;
  if (want < grid) grid = (int)(want < 1 ? 1 : want);
  // work: FL_PCG_WORK doubles, zero-initialised once by the caller; block
  // partials at the front, the completion counter in the last slot
  PhaseArgs a{b, x, r, p, A, P, N, s, work, out, reinterpret_cast<unsigned*>(work + FL_PCG_WORK - 1)};
  if (which == 0) k_pcg_init<<<grid, PCG_NT, 0, st>>>(a);
  if (which == 1) k_pcg_update<<<grid, PCG_NT, 0, st>>>(a);
  if (which == 2) k_pcg_direction<<<grid, PCG_NT, 0, st>>>(a);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

}  // namespace fl
