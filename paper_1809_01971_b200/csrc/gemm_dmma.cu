// Strided batched FP64 GEMM on the tensor cores (DMMA), hand-written.
//
// Used by the dense sine-matrix DST-I (lengths without an FFT plan: the
// reference's dst_apply falls back to the dense orthonormal sine matrix for
// them, spectral.py:163-186) and by the dense eigenbasis transforms of
// generalized modes (spectral.py:122-150's Q / Q^T).  tcgen05 has no f64
// kind, so the FP64 tensor path on sm_100a is mma.sync m8n8k4 (SASS DMMA).
//
//   C[b] = alpha * (A[b] B[b]) (.* E[b]) + beta * C[b]
//
// with arbitrary element strides on every operand (row- or column-major A,
// B, C; batch strides may be 0) and an optional elementwise epilogue factor
// E that shares C's strides (the core of a dense F diag(core) F sandwich).
//
// CTA tile 64 x 64, K step 16, 4 warps in a 2 x 2 arrangement, each warp a
// 32 x 32 sub-tile = 4 x 4 m8n8k4 fragments (32 accumulator doubles per
// lane).  Operand tiles are loaded global -> registers -> shared memory with
// the thread mapping chosen so that consecutive threads walk the operand's
// unit-stride dimension (coalesced for every layout the callers use), and
// the next K tile is held in registers while the current one is consumed
// (one shared buffer, two barriers per K step).  Shared-memory padding makes
// both fragment gathers two wavefronts per warp (the minimum for 256 B).
#include "common.cuh"
#include "kernels.cuh"

namespace fl {
namespace {

constexpr int GBM = 64, GBN = 64, GBK = 16, GNT = 128;
constexpr int AS_LD = GBK + 4;  // As[m][k]: 20-double rows (k gathers: 8 rows x 4 cols, 2 wavefronts)
constexpr int BS_LD = GBN + 8;  // Bs[k][n]: 72-double rows (4 rows x 8 cols, 2 wavefronts)

struct DmmaArgs {
  int64_t M, N, K;
  double alpha, beta;
  const double* A;
  int64_t sAm, sAk, bA;
  const double* B;
  int64_t sBk, sBn, bB;
  double* C;
  int64_t sCm, sCn, bC;
  const double* E;  // optional epilogue factor with C's strides
  int64_t nfast;    // tiles of the faster-varying grid dimension
  int n_fast;       // 1: N tiles vary fastest along blockIdx.x, 0: M tiles
};

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool A_KMAJOR, bool B_NMAJOR>
__global__ void __launch_bounds__(GNT) k_gemm_dmma(const DmmaArgs g) {
  __shared__ double As[GBM * AS_LD];
  __shared__ double Bs[GBK * BS_LD];
  const int64_t b = blockIdx.z;
  const double* __restrict__ A = g.A + b * g.bA;
  const double* __restrict__ B = g.B + b * g.bB;
  // linear tile index, the operand dimension with fewer tiles fastest: the
  // CTAs that run together share the slab of the larger operand (one DRAM
  // read, then L2 hits)
  const int64_t tl = blockIdx.x, tf = tl % g.nfast, ts = tl / g.nfast;
  const int64_t m0 = (g.n_fast ? ts : tf) * GBM, n0 = (g.n_fast ? tf : ts) * GBN;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;

  // tile element e = t + GNT * r (r < 8) of the 64 x 16 A tile / 16 x 64 B tile
  auto a_idx = [&](int e, int& mm, int& kk) {
    if (A_KMAJOR) {
      kk = e & (GBK - 1);
      mm = e >> 4;
    } else {
      mm = e & (GBM - 1);
      kk = e >> 6;
    }
  };
  auto b_idx = [&](int e, int& kb, int& nn) {
    if (B_NMAJOR) {
      nn = e & (GBN - 1);
      kb = e >> 6;
    } else {
      kb = e & (GBK - 1);
      nn = e >> 4;
    }
  };
  double ra[8], rb[8];
  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int mm, kk, kb, nn;
      a_idx(t + GNT * r, mm, kk);
      b_idx(t + GNT * r, kb, nn);
      const int64_t gm = m0 + mm, gk = k0 + kk, gn = n0 + nn, gkb = k0 + kb;
      ra[r] = (gm < g.M && gk < g.K) ? __ldg(A + gm * g.sAm + gk * g.sAk) : 0.0;
      rb[r] = (gn < g.N && gkb < g.K) ? __ldg(B + gkb * g.sBk + gn * g.sBn) : 0.0;
    }
  };
  auto store_tile = [&]() {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int mm, kk, kb, nn;
      a_idx(t + GNT * r, mm, kk);
      b_idx(t + GNT * r, kb, nn);
      As[mm * AS_LD + kk] = ra[r];
      Bs[kb * BS_LD + nn] = rb[r];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;

  // fragment coordinates (m8n8k4, f64): A[row = lane/4][k = lane%4],
  // B[k = lane%4][col = lane/4], C[row = lane/4][col = 2 (lane%4) + {0, 1}]
  const int fr = lane >> 2, fk = lane & 3;
  load_tile(0);
  for (int64_t k0 = 0; k0 < g.K; k0 += GBK) {
    __syncthreads();  // the previous tile has been consumed
    store_tile();
    __syncthreads();
    if (k0 + GBK < g.K) load_tile(k0 + GBK);  // in flight during the MMAs below
#pragma unroll
    for (int ks = 0; ks < GBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[(wm + 8 * i + fr) * AS_LD + ks + fk];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[(ks + fk) * BS_LD + wn + 8 * j + fr];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }

  double* C = g.C + b * g.bC;
  const double* E = g.E ? g.E + b * g.bC : nullptr;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + wm + 8 * i + fr;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int64_t gn = n0 + wn + 8 * j + 2 * fk + h;
        if (gn >= g.N) continue;
        const int64_t off = gm * g.sCm + gn * g.sCn;
        double v = g.alpha * acc[i][j][h];
        if (E) v *= E[off];
        C[off] = (g.beta == 0.0) ? v : fma(g.beta, C[off], v);
      }
    }
  }
}

}  // namespace

int gemm_f64_ep(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sAm, int64_t sAk,
                int64_t bA, const double* B, int64_t sBk, int64_t sBn, int64_t bB, double beta, double* C,
                int64_t sCm, int64_t sCn, int64_t bC, int64_t batch, const double* E, cudaStream_t st) {
  FL_ARG_CHECK(M >= 0 && N >= 0 && K >= 0 && batch >= 0, "bad GEMM shape");
  if (M == 0 || N == 0 || batch == 0) return FL_OK;
  if (N == 1 && bA == 0 && batch > 1) {
    // a batch of matrix-vector products with a shared A is one GEMM:
    // C'[b, m] = sum_k B[b][k] A[m, k]  (M' = batch, N' = M)
    return gemm_f64_ep(batch, M, K, alpha, B, bB, sBk, 0, A, sAk, sAm, 0, beta, C, bC, sCm, 0, 1, E, st);
  }
  const int64_t mt = (M + GBM - 1) / GBM, nt = (N + GBN - 1) / GBN;
  FL_ARG_CHECK(batch <= 65535 && mt * nt < ((int64_t)1 << 31), "GEMM grid too large (M %lld, N %lld, batch %lld)",
               (long long)M, (long long)N, (long long)batch);
  const int n_fast = nt <= mt ? 1 : 0;
  DmmaArgs g{M, N, K, alpha, beta, A, sAm, sAk, bA, B, sBk, sBn, bB, C, sCm, sCn, bC, E, n_fast ? nt : mt, n_fast};
  const dim3 grid((unsigned)(mt * nt), 1u, (unsigned)batch);
  const bool ak = (sAk == 1), bn = (sBn == 1);
  if (ak && bn)
    k_gemm_dmma<true, true><<<grid, GNT, 0, st>>>(g);
  else if (ak)
    k_gemm_dmma<true, false><<<grid, GNT, 0, st>>>(g);
  else if (bn)
    k_gemm_dmma<false, true><<<grid, GNT, 0, st>>>(g);
  else
    k_gemm_dmma<false, false><<<grid, GNT, 0, st>>>(g);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

int gemm_f64(int64_t M, int64_t N, int64_t K, double alpha, const double* A, int64_t sAm, int64_t sAk,
             int64_t bA, const double* B, int64_t sBk, int64_t sBn, int64_t bB, double beta, double* C,
             int64_t sCm, int64_t sCn, int64_t bC, int64_t batch, cudaStream_t st) {
  return gemm_f64_ep(M, N, K, alpha, A, sAm, sAk, bA, B, sBk, sBn, bB, beta, C, sCm, sCn, bC, batch, nullptr, st);
}

}  // namespace fl
