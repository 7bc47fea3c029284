// FFT-based orthonormal DST-I along the middle axis of [outer][n][inner] fp64
// arrays, N = n + 1 a power of two (4 .. 8192).
//
// Algorithm (per tile of C = 2*NFFT lines, all in shared memory):
//   1. load + pre-process (fused): y_j = s_j (x_j + x_{N-j}) + (x_j - x_{N-j})/2,
//      y_{N-j} = s_j (x_j + x_{N-j}) - (x_j - x_{N-j})/2, s_j = sin(pi j / N),
//      y_0 = 0, y_{N/2} = 2 x_{N/2}.  Lines 2p and 2p+1 become the real and
//      imaginary parts of complex sequence p (two real FFTs for the price of one).
//   2. complex DIF FFT of length N in place, radix-8 stages (+ one radix-2/4),
//      output in digit-reversed order (perm table maps frequency -> cell).
//   3. post-process: split the packed spectra, Y^a_k = (C_k + conj C_{N-k})/2,
//      Y^b_k = (C_k - conj C_{N-k})/(2i); even outputs S_{2k} = -Im Y_k, odd
//      outputs S_{2k+1} = Re Y_0/2 + sum_{m=1..k} Re Y_m (segmented scan).
//   4. store (or, for the fused operator pass, scale by the core tensor and run
//      steps 1-3 a second time before storing).
// Shared-memory layout: complex cells [pos][p], p (the FFT index within the
// tile) fastest, XOR-swizzled on p by a fold of pos so that every access
// pattern (row stores, strided butterflies, digit-reversed reads) stays close
// to conflict-free.
#pragma once

#include "common.cuh"

namespace fl {

enum { LOAD_PLAIN = 0, LOAD_KR = 1 };

struct DstArgs {
  const double* x;
  double* y;
  int64_t outer, n, inner;  // x viewed as [outer][n][inner]
  int64_t ntiles, nchunks;  // strided: nchunks = ceil(inner / C)
  double scale;             // applied at the final store
  const double* core;       // fused pass: core tensor, same layout as x
  // LOAD_KR: virtual input Z[j][c] = U[j][c / S] * Xs[j][c % S], inner = R*S
  const double* U;
  const double* Xs;
  int64_t R, S;
  // per-N tables
  const double2* tw;  // N twiddles exp(-2 pi i m / N)
  const double* sn;   // N/2 + 1 values sin(pi j / N)
  const int* perm;    // N: frequency -> cell position
};

template <int LOGN>
struct FftPlan {
  static constexpr int N = 1 << LOGN;
  static constexpr int NST = (LOGN + 2) / 3;
  static constexpr int rlog(int s) { return s < LOGN / 3 ? 3 : LOGN % 3; }
};

template <int LOGF>
__device__ __forceinline__ int swz_key(int pos) {
  if constexpr (LOGF == 0) {
    return 0;
  } else {
    int k = 0;
#pragma unroll
    for (int sh = 0; sh < 14; sh += LOGF) k ^= (pos >> sh);
    return k & ((1 << LOGF) - 1);
  }
}

template <int NFFT>
struct Cells {
  static constexpr int LOGF = NFFT == 1 ? 0 : NFFT == 2 ? 1 : NFFT == 4 ? 2 : NFFT == 8 ? 3 : 4;
  double2* D;
  __device__ __forceinline__ int idx(int pos, int p) const { return pos * NFFT + (p ^ swz_key<LOGF>(pos)); }
  __device__ __forceinline__ double2 ld(int pos, int p) const { return D[idx(pos, p)]; }
  __device__ __forceinline__ void st(int pos, int p, double2 v) const { D[idx(pos, p)] = v; }
  // real element (line l, row j)
  __device__ __forceinline__ double& re(int l, int j) const {
    return reinterpret_cast<double*>(D)[2 * idx(j, l >> 1) + (l & 1)];
  }
};

// ---- small DFTs (forward, e^{-2 pi i tq / R}) ----------------------------
__device__ __forceinline__ void dft2(double2& a0, double2& a1) {
  double2 t = a0;
  a0 = cadd(t, a1);
  a1 = csub(t, a1);
}

__device__ __forceinline__ void dft4(double2& a0, double2& a1, double2& a2, double2& a3) {
  double2 t0 = cadd(a0, a2), t1 = csub(a0, a2);
  double2 t2 = cadd(a1, a3), t3 = cmul_mi(csub(a1, a3));
  a0 = cadd(t0, t2);
  a2 = csub(t0, t2);
  a1 = cadd(t1, t3);
  a3 = csub(t1, t3);
}

__device__ __forceinline__ void dft8(double2 (&a)[8]) {
  constexpr double r = 0.70710678118654752440084436210485;
  dft4(a[0], a[2], a[4], a[6]);  // E0..E3 in a0,a2,a4,a6
  dft4(a[1], a[3], a[5], a[7]);  // O0..O3 in a1,a3,a5,a7
  double2 o1 = a[3], o2 = a[5], o3 = a[7];
  o1 = make_double2((o1.x + o1.y) * r, (o1.y - o1.x) * r);  // * (1 - i)/sqrt2
  o2 = cmul_mi(o2);                                         // * -i
  o3 = make_double2((o3.y - o3.x) * r, -(o3.x + o3.y) * r); // * (-1 - i)/sqrt2
  double2 e0 = a[0], e1 = a[2], e2 = a[4], e3 = a[6], o0 = a[1];
  a[0] = cadd(e0, o0);
  a[4] = csub(e0, o0);
  a[1] = cadd(e1, o1);
  a[5] = csub(e1, o1);
  a[2] = cadd(e2, o2);
  a[6] = csub(e2, o2);
  a[3] = cadd(e3, o3);
  a[7] = csub(e3, o3);
}

template <int RL>
__device__ __forceinline__ void dftR(double2 (&a)[1 << RL]) {
  if constexpr (RL == 1) dft2(a[0], a[1]);
  if constexpr (RL == 2) dft4(a[0], a[1], a[2], a[3]);
  if constexpr (RL == 3) dft8(a);
}

// one DIF stage: sub-length L = 2^LGL, radix R = 2^RL, stride st = L / R
template <int LOGN, int NFFT, int NT, int LGL, int RL>
__device__ __forceinline__ void fft_stage(const Cells<NFFT>& cs, const double2* __restrict__ tw) {
  constexpr int N = 1 << LOGN;
  constexpr int R = 1 << RL;
  constexpr int LGST = LGL - RL;
  constexpr int ST = 1 << LGST;
  constexpr int NB = NFFT * (N / R);  // butterflies in this stage
  constexpr int PER = (NB + NT - 1) / NT;
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int b = threadIdx.x + it * NT;
    if (NB % NT == 0 || b < NB) {
      const int p = b % NFFT;
      const int bi = b / NFFT;
      const int j = bi & (ST - 1);
      const int base = ((bi >> LGST) << LGL) + j;
      double2 v[R];
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = cs.ld(base + t * ST, p);
      dftR<RL>(v);
      if constexpr (LGST > 0) {
#pragma unroll
        for (int q = 1; q < R; ++q) {
          const double2 w = __ldg(&tw[(j * q) << (LOGN - LGL)]);
          v[q] = cmul(v[q], w);
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) cs.st(base + q * ST, p, v[q]);
    }
  }
  __syncthreads();
}

template <int LOGN, int NFFT, int NT, int S, int LGL>
__device__ __forceinline__ void fft_rec(const Cells<NFFT>& cs, const double2* __restrict__ tw) {
  if constexpr (S < FftPlan<LOGN>::NST) {
    constexpr int RL = FftPlan<LOGN>::rlog(S);
    fft_stage<LOGN, NFFT, NT, LGL, RL>(cs, tw);
    fft_rec<LOGN, NFFT, NT, S + 1, LGL - RL>(cs, tw);
  }
}

// exclusive scan of v over aligned groups of G consecutive threads
template <int G, int NT>
__device__ __forceinline__ double2 group_excl_scan(double2 v, double* scr) {
  constexpr int W = G < 32 ? G : 32;
  const int lane = threadIdx.x & 31;
  double2 x = v;
#pragma unroll
  for (int d = 1; d < W; d <<= 1) {
    const double yx = __shfl_up_sync(0xffffffffu, x.x, d, W);
    const double yy = __shfl_up_sync(0xffffffffu, x.y, d, W);
    if ((lane & (W - 1)) >= d) {
      x.x += yx;
      x.y += yy;
    }
  }
  if constexpr (G <= 32) {
    return make_double2(x.x - v.x, x.y - v.y);
  } else {
    const int warp = threadIdx.x >> 5;
    if (lane == 31) {
      scr[2 * warp] = x.x;
      scr[2 * warp + 1] = x.y;
    }
    __syncthreads();
    constexpr int WPG = G / 32;
    const int first = (warp / WPG) * WPG;
    double ox = 0.0, oy = 0.0;
    for (int w = first; w < warp; ++w) {
      ox += scr[2 * w];
      oy += scr[2 * w + 1];
    }
    __syncthreads();
    return make_double2(x.x - v.x + ox, x.y - v.y + oy);
  }
}

// post-process the packed spectra into natural-order DST outputs (times sc)
template <int LOGN, int NFFT, int NT>
__device__ __forceinline__ void dst_post(const Cells<NFFT>& cs, const int* __restrict__ perm,
                                         double sc, double* scr) {
  constexpr int N = 1 << LOGN;
  constexpr int H = N / 2;
  constexpr int G0 = NT / NFFT;
  constexpr int G = G0 < H ? G0 : H;
  constexpr int KPT = H / G;
  const int t = threadIdx.x;
  const bool active = t < NFFT * G;
  const int p = t / G;
  const int g = t % G;
  double ea[KPT], eb[KPT], oa[KPT], ob[KPT];
  double2 tot = make_double2(0.0, 0.0);
  if (active) {
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = g * KPT + i;
      const double2 ck = cs.ld(__ldg(&perm[k]), p);
      const double2 cm = cs.ld(__ldg(&perm[(N - k) & (N - 1)]), p);
      ea[i] = 0.5 * (cm.y - ck.y);
      eb[i] = 0.5 * (ck.x - cm.x);
      double ra = 0.5 * (ck.x + cm.x);
      double rb = 0.5 * (ck.y + cm.y);
      if (k == 0) {
        ra *= 0.5;
        rb *= 0.5;
      }
      tot.x += ra;
      tot.y += rb;
      oa[i] = tot.x;
      ob[i] = tot.y;
    }
  }
  const double2 off = group_excl_scan<G, NT>(active ? tot : make_double2(0.0, 0.0), scr);
  __syncthreads();
  if (active) {
#pragma unroll
    for (int i = 0; i < KPT; ++i) {
      const int k = g * KPT + i;
      cs.st(2 * k, p, make_double2(ea[i] * sc, eb[i] * sc));
      cs.st(2 * k + 1, p, make_double2((oa[i] + off.x) * sc, (ob[i] + off.y) * sc));
    }
  }
  __syncthreads();
}

template <bool CONTIG, int C>
__device__ __forceinline__ bool line_ok(const DstArgs& a, int64_t tile, int l, int64_t& off0, int64_t& jstride) {
  if (CONTIG) {
    const int64_t L = tile * C + l;
    off0 = L * a.n;
    jstride = 1;
    return L < a.outer;
  } else {
    const int64_t o = tile / a.nchunks;
    const int64_t c = (tile % a.nchunks) * C + l;
    off0 = o * a.n * a.inner + c;
    jstride = a.inner;
    return c < a.inner;
  }
}

template <int LOADER>
__device__ __forceinline__ double load_elem(const DstArgs& a, int64_t off0, int64_t row, int64_t jstride) {
  if constexpr (LOADER == LOAD_PLAIN) {
    return __ldg(&a.x[off0 + row * jstride]);
  } else {
    // off0 == c (column of the virtual R*S matrix, outer == 1), jstride == R*S
    const int64_t c = off0;
    const int64_t k = c / a.S, s = c - k * a.S;
    return __ldg(&a.U[row * a.R + k]) * __ldg(&a.Xs[row * a.S + s]);
  }
}

// stage 1: global -> smem with the DST-I pre-processing fused in.
// MODE 0: load from x; MODE 1: smem already holds a transform, scale by core.
template <bool CONTIG, int C, int H>
__device__ __forceinline__ void item_lj(int item, int& l, int& jj) {
  if (CONTIG) {
    l = item / H;
    jj = item % H;
  } else {
    l = item % C;
    jj = item / C;
  }
}

template <int LOGN, int NFFT, int NT, bool CONTIG, int LOADER, int MODE>
__device__ __forceinline__ void dst_pre(const DstArgs& a, const Cells<NFFT>& cs, int64_t tile) {
  constexpr int N = 1 << LOGN;
  constexpr int H = N / 2;
  constexpr int C = 2 * NFFT;
  constexpr int ITEMS = C * H;
  constexpr int PER = (ITEMS + NT - 1) / NT;
  constexpr int B = PER < 4 ? PER : 4;  // items whose loads are batched
  static_assert(PER % B == 0, "batch must divide the per-thread item count");
  for (int it0 = 0; it0 < PER; it0 += B) {
    double xa[B], xb[B];
    bool ok[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int item = threadIdx.x + (it0 + u) * NT;
      int l, jj;
      item_lj<CONTIG, C, H>(item, l, jj);
      const int j = jj + 1;
      int64_t off0, js;
      ok[u] = (ITEMS % NT == 0 || item < ITEMS) && line_ok<CONTIG, C>(a, tile, l, off0, js);
      xa[u] = 0.0;
      xb[u] = 0.0;
      if (MODE == 0) {
        if (ok[u]) {
          xa[u] = load_elem<LOADER>(a, off0, j - 1, js);
          if (j < H) xb[u] = load_elem<LOADER>(a, off0, N - j - 1, js);
        }
      } else if (ok[u]) {
        xa[u] = __ldg(&a.core[off0 + (int64_t)(j - 1) * js]);
        if (j < H) xb[u] = __ldg(&a.core[off0 + (int64_t)(N - j - 1) * js]);
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int item = threadIdx.x + (it0 + u) * NT;
      if (ITEMS % NT == 0 || item < ITEMS) {
        int l, jj;
        item_lj<CONTIG, C, H>(item, l, jj);
        const int j = jj + 1;
        double va = xa[u], vb = xb[u];
        if (MODE == 1) {
          // xa/xb hold core values; scale the forward transform held in smem
          va = ok[u] ? cs.re(l, j) * va : 0.0;
          vb = (ok[u] && j < H) ? cs.re(l, N - j) * vb : 0.0;
        }
        if (j == H) {
          cs.re(l, H) = 2.0 * va;
        } else {
          const double s = __ldg(&a.sn[j]);
          const double sum = s * (va + vb), dif = 0.5 * (va - vb);
          cs.re(l, j) = sum + dif;
          cs.re(l, N - j) = sum - dif;
        }
      }
    }
  }
  if (MODE == 0) {
    for (int l = threadIdx.x; l < C; l += NT) cs.re(l, 0) = 0.0;
  }
}

template <int LOGN, int NFFT, int NT, bool CONTIG>
__device__ __forceinline__ void dst_store(const DstArgs& a, const Cells<NFFT>& cs, int64_t tile) {
  constexpr int N = 1 << LOGN;
  constexpr int C = 2 * NFFT;
  constexpr int ROWS = N - 1;
  constexpr int ITEMS = C * ROWS;
  constexpr int PER = (ITEMS + NT - 1) / NT;
#pragma unroll 4
  for (int it = 0; it < PER; ++it) {
    const int item = threadIdx.x + it * NT;
    if (item < ITEMS) {
      int l, j;
      if (CONTIG) {
        l = item / ROWS;
        j = item % ROWS + 1;
      } else {
        l = item % C;
        j = item / C + 1;
      }
      int64_t off0, js;
      if (line_ok<CONTIG, C>(a, tile, l, off0, js)) a.y[off0 + (int64_t)(j - 1) * js] = cs.re(l, j);
    }
  }
}

template <int LOGN, int NFFT, int NT, int MINB, bool CONTIG, int LOADER, bool MIDCORE>
__global__ void __launch_bounds__(NT, MINB) k_dst_fft(const DstArgs a) {
  extern __shared__ __align__(16) double smem_dst[];
  Cells<NFFT> cs{reinterpret_cast<double2*>(smem_dst)};
  double* scr = smem_dst + 2 * (1 << LOGN) * NFFT;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    dst_pre<LOGN, NFFT, NT, CONTIG, LOADER, 0>(a, cs, tile);
    __syncthreads();
    fft_rec<LOGN, NFFT, NT, 0, LOGN>(cs, a.tw);
    if constexpr (MIDCORE) {
      dst_post<LOGN, NFFT, NT>(cs, a.perm, 1.0, scr);
      dst_pre<LOGN, NFFT, NT, CONTIG, LOADER, 1>(a, cs, tile);
      __syncthreads();
      fft_rec<LOGN, NFFT, NT, 0, LOGN>(cs, a.tw);
    }
    dst_post<LOGN, NFFT, NT>(cs, a.perm, a.scale, scr);
    dst_store<LOGN, NFFT, NT, CONTIG>(a, cs, tile);
    __syncthreads();
  }
}

// launch-shape policy per transform length: <= 64 registers per thread,
// >= 32 resident warps per SM where shared memory allows
template <int LOGN>
struct DstShape {
  static constexpr int NFFT = LOGN <= 8 ? 16 : (LOGN >= 12 ? 1 : (8 >> (LOGN - 9)));
  static constexpr int NT = LOGN >= 13 ? 1024 : (LOGN >= 8 ? 512 : (LOGN <= 5 ? 128 : 256));
  static constexpr int MINB = LOGN >= 13 ? 1 : (LOGN >= 8 ? 2 : (LOGN <= 5 ? 8 : 4));
  static constexpr size_t SMEM = size_t(16) * (size_t(1) << LOGN) * NFFT + size_t(16) * (NT / 32);
};

}  // namespace fl
