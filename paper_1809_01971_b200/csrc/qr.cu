// R factor of tall-skinny QR factorisations by communication-avoiding
// Householder QR (TSQR), for the truncation's factor SVDs (decomp.py:343-345,
// 373, 395: SVDs of n x R factor matrices with n <= 128 << R).  The wide
// matrix M (k x m, k <= 128) has the left singular system of the k x k
// triangle R of M^T = Q R, so the long side is reduced here and the small
// factor goes to the one-CTA pivoted Jacobi (svd.cu).
//
// Leaves: CTA (g, i) owns a slice of M_i's columns (= rows of M_i^T), keeps
// its k x k triangle in shared memory and absorbs the slice in chunks of 128
// rows held in registers (absorb_chunk below).  Tree: pairs of triangles are
// merged the same way (the second triangle is the chunk), one launch per
// level; the result lands in slot 0.  The critical path is (chunks per leaf
// + levels) x k Householder steps of ~0.25 us.
#include <climits>
#include "common.cuh"
#include "kernels.cuh"

namespace fl {

namespace {

constexpr int TS_THREADS = 512;
constexpr int TS_CHUNK = 128;  // rows absorbed per phase

// One phase: the CTA holds R (k x k, row-major in shared memory) and absorbs
// a chunk of up to TS_CHUNK rows that lives in REGISTERS: LPC lanes per
// column, lane q of column c holds chunk rows q, q + LPC, ...  Step j: the
// lanes of column j form the reflector (diagonal entry + their chunk column),
// publish it (double-buffered by step parity: one CTA barrier per step), and
// the lanes of the columns c > j apply it to R[j][c] and to their registers.
// Shared-memory traffic per step is the reflector only; the chunk is never
// written back.
template <int LPC>
__device__ __forceinline__ void absorb_chunk(double* Rs, int ldr, double* vbuf, double* sc, int k, bool tri,
                                             double (&x)[TS_CHUNK / LPC]) {
  constexpr int RPT = TS_CHUNK / LPC;
  const int c = threadIdx.x / LPC, q = threadIdx.x % LPC;
  const unsigned gmask = (LPC == 32 ? 0xffffffffu : ((1u << LPC) - 1u)) << ((threadIdx.x & 31) & ~(LPC - 1));
  for (int j = 0; j < k; ++j) {
    double* vb = vbuf + (j & 1) * TS_CHUNK;
    double* scj = sc + (j & 1) * 2;
    if (c == j) {
      double s0 = 0.0, s1 = 0.0;
#pragma unroll
      for (int i = 0; i < RPT; i += 2) {
        s0 = fma(x[i], x[i], s0);
        s1 = fma(x[i + 1], x[i + 1], s1);
      }
      double s = s0 + s1;
#pragma unroll
      for (int o = 1; o < LPC; o <<= 1) s += __shfl_xor_sync(gmask, s, o);
      const double xj = Rs[(size_t)j * ldr + j];
      double alpha = xj, v0 = 0.0, beta = 0.0;
      if (s > 0.0) {
        alpha = -copysign(sqrt(fma(xj, xj, s)), xj);
        v0 = xj - alpha;
        beta = 2.0 / fma(v0, v0, s);
      }
#pragma unroll
      for (int i = 0; i < RPT; ++i) vb[q + LPC * i] = x[i];
      if (q == 0) {
        scj[0] = v0;
        scj[1] = beta;
        Rs[(size_t)j * ldr + j] = alpha;
      }
    }
    __syncthreads();
    const double beta = scj[1];
    if (beta != 0.0 && c > j && c < k) {
      const double v0 = scj[0];
      // reflector entries are re-read in blocks of 8 (the chunk already
      // takes 2 * RPT registers; a compiler fence keeps a block's loads from
      // being hoisted over the previous block)
      const double rjc = Rs[(size_t)j * ldr + c];
      double d0 = 0.0, d1 = 0.0;
#pragma unroll
      for (int i0 = 0; i0 < RPT; i0 += 8) {
        if (tri && LPC * i0 > j) break;  // merge: the reflector is zero below chunk row j
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = vb[q + LPC * (i0 + i)];
#pragma unroll
        for (int i = 0; i < 8; i += 2) {
          d0 = fma(v[i], x[i0 + i], d0);
          d1 = fma(v[i + 1], x[i0 + i + 1], d1);
        }
        asm volatile("" ::: "memory");
      }
      double d = d0 + d1;
#pragma unroll
      for (int o = 1; o < LPC; o <<= 1) d += __shfl_xor_sync(gmask, d, o);
      d = fma(v0, rjc, d) * beta;
#pragma unroll
      for (int i0 = 0; i0 < RPT; i0 += 8) {
        if (tri && LPC * i0 > j) break;  // merge: the reflector is zero below chunk row j
        double v[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) v[i] = vb[q + LPC * (i0 + i)];
#pragma unroll
        for (int i = 0; i < 8; ++i) x[i0 + i] = fma(-d, v[i], x[i0 + i]);
        asm volatile("" ::: "memory");
      }
      if (q == 0) Rs[(size_t)j * ldr + c] = fma(-d, v0, rjc);
    }
  }
}

struct TsqrBatch {
  const double* src[FL_QR_MAX_BATCH];
  double* slot0[FL_QR_MAX_BATCH];  // k x k row-major: the result
  double* ws[FL_QR_MAX_BATCH];     // slots 1 .. leaves-1
  long long rs[FL_QR_MAX_BATCH], cs[FL_QR_MAX_BATCH], m[FL_QR_MAX_BATCH];
  int k[FL_QR_MAX_BATCH], leaves[FL_QR_MAX_BATCH];
};

__device__ __forceinline__ double* ts_slot(const TsqrBatch& tb, int i, int g) {
  const size_t kk = (size_t)tb.k[i] * tb.k[i];
  return g == 0 ? tb.slot0[i] : tb.ws[i] + (size_t)(g - 1) * kk;
}

template <int LPC>
__device__ __forceinline__ void tsqr_cta(const TsqrBatch& tb, int stride, double* Rs, double* vbuf, double* sc) {
  constexpr int RPT = TS_CHUNK / LPC;
  const int i = blockIdx.y, g = blockIdx.x;
  const int k = tb.k[i], G = tb.leaves[i], ldr = k;
  const int c = threadIdx.x / LPC, q = threadIdx.x % LPC;
  double x[RPT];
  int slot;
  if (stride == 0) {
    if (g >= G) return;
    slot = g;
    const long long m = tb.m[i], rs = tb.rs[i], cs = tb.cs[i];
    const long long per = (m + G - 1) / G;
    const long long c_lo = (long long)g * per, c_hi = min(m, c_lo + per);
    const double* M = tb.src[i];
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) Rs[idx] = 0.0;
    __syncthreads();
    for (long long pos = c_lo; pos < c_hi; pos += TS_CHUNK) {
#pragma unroll
      for (int t = 0; t < RPT; ++t) {
        const long long col = pos + q + LPC * t;
        x[t] = (c < k && col < c_hi) ? M[c * rs + col * cs] : 0.0;
      }
      absorb_chunk<LPC>(Rs, ldr, vbuf, sc, k, false, x);
    }
  } else {
    const int a = 2 * stride * g, b = a + stride;
    if (b >= G) return;
    slot = a;
    const double* Ra = ts_slot(tb, i, a);
    const double* Rb = ts_slot(tb, i, b);
    for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) Rs[idx] = Ra[idx];
#pragma unroll
    for (int t = 0; t < RPT; ++t) {
      const int row = q + LPC * t;
      x[t] = (c < k && row < k && row <= c) ? Rb[(size_t)row * k + c] : 0.0;
    }
    __syncthreads();
    absorb_chunk<LPC>(Rs, ldr, vbuf, sc, k, true, x);
  }
  __syncthreads();
  double* out = ts_slot(tb, i, slot);
  for (int idx = threadIdx.x; idx < k * k; idx += blockDim.x) {
    const int r = idx / k, cc = idx - r * k;
    out[idx] = cc >= r ? Rs[idx] : 0.0;
  }
}

// stride == 0: leaves; stride = s > 0: merge slots a = 2 s g and a + s into a
__global__ void __launch_bounds__(TS_THREADS, 1) k_tsqr(const TsqrBatch tb, int stride) {
  extern __shared__ double sm_ts[];
  const int k = tb.k[blockIdx.y];
  double* Rs = sm_ts;
  double* vbuf = sm_ts + (size_t)k * k;
  double* sc = vbuf + 2 * TS_CHUNK;
  if (k <= 32)
    tsqr_cta<16>(tb, stride, Rs, vbuf, sc);
  else if (k <= 64)
    tsqr_cta<8>(tb, stride, Rs, vbuf, sc);
  else
    tsqr_cta<4>(tb, stride, Rs, vbuf, sc);
}

}  // namespace

// R_i (k_i x k_i row-major, upper triangular) of M_i^T = Q R for a batch of
// wide matrices M_i (k_i x m_i, element (r, c) at M_i[r * rs_i + c * cs_i]).
int tsqr_r(int batch, const double* const* M, const int* k, const int64_t* m, const int64_t* rs, const int64_t* cs,
           double* const* R, cudaStream_t st) {
  FL_ARG_CHECK(batch >= 0 && batch <= FL_QR_MAX_BATCH, "TSQR batch must be 0..%d", FL_QR_MAX_BATCH);
  if (batch == 0) return FL_OK;
  TsqrBatch tb{};
  int gmax = 1;
  size_t ws_total = 0, smem = 0;
  size_t ws_off[FL_QR_MAX_BATCH];
  for (int i = 0; i < batch; ++i) {
    FL_ARG_CHECK(k[i] >= 1 && k[i] <= FL_QR_MAX_K, "TSQR: k = %d outside 1..%d", k[i], FL_QR_MAX_K);
    FL_ARG_CHECK(m[i] >= 1, "TSQR: empty matrix");
    FL_ARG_CHECK(M[i] != nullptr && R[i] != nullptr, "TSQR: null matrix");
    // phases on the critical path: chunks per leaf + merge levels; take the
    // power-of-two leaf count that minimises them
    int G = 1, best = INT_MAX;
    for (int cand = 1, lev = 0; cand <= FL_QR_MAX_LEAVES; cand *= 2, ++lev) {
      const int64_t per = (m[i] + cand - 1) / cand;
      if (cand > 1 && per < TS_CHUNK / 2) break;
      const int cost = (int)((per + TS_CHUNK - 1) / TS_CHUNK) + lev;
      if (cost < best) {
        best = cost;
        G = cand;
      }
    }
    const int64_t per = (m[i] + G - 1) / G;
    G = (int)((m[i] + per - 1) / per);  // no empty leaves
    tb.src[i] = M[i];
    tb.slot0[i] = R[i];
    tb.rs[i] = rs[i];
    tb.cs[i] = cs[i];
    tb.m[i] = m[i];
    tb.k[i] = k[i];
    tb.leaves[i] = G;
    ws_off[i] = ws_total;
    ws_total += (size_t)(G - 1) * k[i] * k[i];
    if (G > gmax) gmax = G;
    const size_t sz = sizeof(double) * ((size_t)k[i] * k[i] + 2 * TS_CHUNK + 4);
    if (sz > smem) smem = sz;
  }
  DevBuf ws;
  if (ws_total) {
    int rc = ws.alloc((int64_t)ws_total, st);
    if (rc) return rc;
  }
  for (int i = 0; i < batch; ++i) tb.ws[i] = ws.p ? ws.p + ws_off[i] : nullptr;
  static unsigned long long attr_done = 0;  // bit per device ordinal
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  const unsigned long long bit = 1ull << (dev & 63);
  if (!(__atomic_load_n(&attr_done, __ATOMIC_ACQUIRE) & bit)) {
    const size_t cap = sizeof(double) * ((size_t)FL_QR_MAX_K * FL_QR_MAX_K + 2 * TS_CHUNK + 4);
    FL_CUDA_TRY(cudaFuncSetAttribute(k_tsqr, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap));
    __atomic_fetch_or(&attr_done, bit, __ATOMIC_RELEASE);
  }
  k_tsqr<<<dim3(gmax, batch), TS_THREADS, smem, st>>>(tb, 0);
  FL_LAUNCH_CHECK();
  for (int s = 1; s < gmax; s *= 2) {
    const int pairs = (gmax + 2 * s - 1) / (2 * s);
    k_tsqr<<<dim3(pairs, batch), TS_THREADS, smem, st>>>(tb, s);
    FL_LAUNCH_CHECK();
  }
  return FL_OK;
}

}  // namespace fl
