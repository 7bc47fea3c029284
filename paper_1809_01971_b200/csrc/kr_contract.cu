// Khatri-Rao contraction on the FP64 tensor cores, hand-written:
//
//   out[(ia, ib), j] = sum_r Pa[ia, r] Pb[ib, r] Y[r, j]
//
// the workhorse of the canonical-to-Tucker ALS (decomp.py:384-399: the
// mode-l matrix U_l (KR(Pa, Pb) diag(xi))^T) and of the core projection
// (decomp.py:349-353).  The (a b) x R Khatri-Rao operand is never formed:
// the A tile of the DMMA GEMM is generated while loading (two coalesced reads
// and a product per element).  a b x N outputs are few tiles (N <= 128 after
// range compression) while R reaches 1e5, so the reduction is split over R:
// split s accumulates its slice into its own partial, and a second kernel
// sums the partials in a fixed order (deterministic, unlike atomics).
//
// Tiling as gemm_dmma.cu: CTA tile 64 x 64, K step 16, 4 warps of 32 x 32
// (mma.sync m8n8k4 f64 = SASS DMMA), register-staged prefetch of the next K
// tile.
#include "common.cuh"
#include "kernels.cuh"

namespace fl {
namespace {

constexpr int KBM = 64, KBN = 64, KBK = 16, KNT = 128;
constexpr int KAS_LD = KBK + 4, KBS_LD = KBN + 8;
// Y with unit stride along r (the transposed view (U diag(xi))^T): the B tile
// is kept n-major like the A tile, so that the threads that walk r in global
// memory also walk it in shared memory (the k-major layout made those stores
// 8-way bank conflicts: 11 instead of ~20 TFLOP/s)
constexpr int KBT_LD = KBK + 4;
constexpr int KB_ELEMS = (KBK * KBS_LD > KBN * KBT_LD) ? KBK * KBS_LD : KBN * KBT_LD;

struct KrArgs {
  const double* Pa;
  const double* Pb;
  const double* Y;
  double* out;      // splits == 1: the result; else partials [split][M][N]
  int64_t a, b, R, N;
  int64_t sYr, sYj;
  int64_t kc;       // reduction indices per split (multiple of KBK)
  int64_t mt, nt;
};

__device__ __forceinline__ void kr_dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <bool Y_JMAJOR>
__global__ void __launch_bounds__(KNT) k_kr_dmma(const KrArgs g) {
  __shared__ double As[KBM * KAS_LD];
  __shared__ double Bs[KB_ELEMS];
  const int64_t M = g.a * g.b;
  const int64_t tl = blockIdx.x, tn = tl % g.nt, tm = tl / g.nt;
  const int64_t m0 = tm * KBM, n0 = tn * KBN;
  const int64_t k_lo = (int64_t)blockIdx.y * g.kc, k_hi = min(g.R, k_lo + g.kc);
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  // A tile element e = t + KNT * r: kk = e & 15 (reduction index, unit
  // stride in Pa / Pb), mm = e >> 4: rows (t >> 4) + 8 r of the tile
  const int akk = t & (KBK - 1);
  // per-thread operand pointers, advanced by one K tile per load (address
  // arithmetic was a third of the instructions with per-load index products)
  const double* pa[8];
  const double* pb[8];
  const double* py[8];
  unsigned okrow = 0, okcol = 0;
#pragma unroll
  for (int r = 0; r < 8; ++r) {
    const int64_t gm = m0 + (t >> 4) + 8 * r;
    pa[r] = g.Pa;
    pb[r] = g.Pb;
    if (gm < M) {
      const int64_t ia = gm / g.b;
      pa[r] = g.Pa + ia * g.R + k_lo + akk;
      pb[r] = g.Pb + (gm - ia * g.b) * g.R + k_lo + akk;
      okrow |= 1u << r;
    }
    const int e = t + KNT * r;
    const int kb = Y_JMAJOR ? (e >> 6) : (e & (KBK - 1));
    const int nn = Y_JMAJOR ? (e & (KBN - 1)) : (e >> 4);
    py[r] = g.Y;
    if (n0 + nn < g.N) {
      py[r] = g.Y + (k_lo + kb) * g.sYr + (n0 + nn) * g.sYj;
      okcol |= 1u << r;
    }
  }
  const int64_t ystep = (int64_t)KBK * g.sYr;
  // raw Pa and Pb values: the product is formed at store time so that the
  // loads stay in flight during the MMAs of the current tile
  double ra[8], rp[8], rb[8];
  auto load_tile = [&](int64_t k0) {
    const int64_t krem = k_hi - k0;  // reduction indices left in this split
    const bool aok = akk < krem;
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      const bool ok = aok && ((okrow >> r) & 1u);
      ra[r] = ok ? __ldg(pa[r]) : 0.0;
      rp[r] = ok ? __ldg(pb[r]) : 0.0;
      pa[r] += KBK;
      pb[r] += KBK;
      const int e = t + KNT * r;
      const int kb = Y_JMAJOR ? (e >> 6) : (e & (KBK - 1));
      rb[r] = (kb < krem && ((okcol >> r) & 1u)) ? __ldg(py[r]) : 0.0;
      py[r] += ystep;
    }
  };
  auto store_tile = [&]() {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      As[((t >> 4) + 8 * r) * KAS_LD + akk] = ra[r] * rp[r];
      const int e = t + KNT * r;
      int kb, nn;
      if (Y_JMAJOR) {
        nn = e & (KBN - 1);
        kb = e >> 6;
      } else {
        kb = e & (KBK - 1);
        nn = e >> 4;
      }
      if (Y_JMAJOR)
        Bs[kb * KBS_LD + nn] = rb[r];
      else
        Bs[nn * KBT_LD + kb] = rb[r];
    }
  };
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  const int fr = lane >> 2, fk = lane & 3;
  if (k_lo < k_hi) load_tile(k_lo);
  for (int64_t k0 = k_lo; k0 < k_hi; k0 += KBK) {
    __syncthreads();
    store_tile();
    __syncthreads();
    if (k0 + KBK < k_hi) load_tile(k0 + KBK);
#pragma unroll
    for (int ks = 0; ks < KBK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[(wm + 8 * i + fr) * KAS_LD + ks + fk];
#pragma unroll
      for (int j = 0; j < 4; ++j)
        bf[j] = Y_JMAJOR ? Bs[(ks + fk) * KBS_LD + wn + 8 * j + fr] : Bs[(wn + 8 * j + fr) * KBT_LD + ks + fk];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) kr_dmma(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
  }
  double* C = g.out + (size_t)blockIdx.y * M * g.N;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int64_t gm = m0 + wm + 8 * i + fr;
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gn = n0 + wn + 8 * j + 2 * fk;
      if (gn < g.N) C[gm * g.N + gn] = acc[i][j][0];
      if (gn + 1 < g.N) C[gm * g.N + gn + 1] = acc[i][j][1];
    }
  }
}

// out[idx] = sum over splits, in split order
__global__ void k_kr_reduce(const double* __restrict__ part, double* __restrict__ out, int64_t count, int splits) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += (int64_t)gridDim.x * blockDim.x) {
    double s = part[i];
    for (int p = 1; p < splits; ++p) s += part[(size_t)p * count + i];
    out[i] = s;
  }
}

}  // namespace

int kr_contract(const double* Pa, int64_t a, const double* Pb, int64_t b, int64_t R, const double* Y, int64_t sYr,
                int64_t sYj, int64_t N, double* out, cudaStream_t st) {
  FL_ARG_CHECK(a >= 1 && b >= 1 && R >= 0 && N >= 1 && a < (1 << 30) && b < (1 << 30), "bad Khatri-Rao contraction shape");
  FL_ARG_CHECK(Pa && Pb && Y && out, "Khatri-Rao contraction: null operand");
  const int64_t M = a * b;
  const int64_t mt = (M + KBM - 1) / KBM, nt = (N + KBN - 1) / KBN;
  FL_ARG_CHECK(mt * nt < ((int64_t)1 << 31), "Khatri-Rao contraction: grid too large");
  if (R == 0) {
    FL_CUDA_TRY(cudaMemsetAsync(out, 0, sizeof(double) * (size_t)M * N, st));
    return FL_OK;
  }
  // split count: whole waves of resident CTAs (the tiles of one problem are
  // few: a ragged last wave cost 28% at 80 tiles x 8 splits), slices of at
  // least 256 reduction indices
  static int per_sm[2] = {0, 0};
  const int var = sYj == 1 ? 0 : 1;
  if (per_sm[var] == 0) {
    int v = 0;
    if (var == 0)
      FL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_kr_dmma<true>, KNT, 0));
    else
      FL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, k_kr_dmma<false>, KNT, 0));
    per_sm[var] = v > 0 ? v : 1;
  }
  const double wave = (double)per_sm[var] * sm_count();
  const int64_t tiles = mt * nt;
  int64_t max_splits = (R + 255) / 256;
  if (max_splits > 64) max_splits = 64;
  int64_t splits = 1;
  double best = -1.0;
  for (int64_t sp = 1; sp <= max_splits; ++sp) {
    const double waves = (double)(tiles * sp) / wave;
    const double full = waves < 1.0 ? 1.0 : (double)(int64_t)(waves + 0.999999);
    // efficiency of the last wave, discounted a little per extra split (the
    // partials are written and summed again)
    const double score = waves / full - 0.004 * (double)sp;
    if (score > best) {
      best = score;
      splits = sp;
    }
  }
  int64_t kc = ((R + splits - 1) / splits + KBK - 1) / KBK * KBK;
  splits = (R + kc - 1) / kc;
  DevBuf part;
  if (splits > 1) {
    int rc = part.alloc(splits * M * N, st);
    if (rc) return rc;
  }
  KrArgs g{Pa, Pb, Y, splits > 1 ? part.p : out, a, b, R, N, sYr, sYj, kc, mt, nt};
  const dim3 grid((unsigned)(mt * nt), (unsigned)splits);
  if (sYj == 1)
    k_kr_dmma<true><<<grid, KNT, 0, st>>>(g);
  else
    k_kr_dmma<false><<<grid, KNT, 0, st>>>(g);
  FL_LAUNCH_CHECK();
  if (splits > 1) {
    const int64_t count = M * N;
    const int blocks = (int)((count + 255) / 256 < 4096 ? (count + 255) / 256 : 4096);
    k_kr_reduce<<<blocks, 256, 0, st>>>(part.p, out, count, (int)splits);
    FL_LAUNCH_CHECK();
  }
  return FL_OK;
}

}  // namespace fl
