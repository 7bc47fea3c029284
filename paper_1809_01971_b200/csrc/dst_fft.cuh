// FFT-based orthonormal DST-I along the middle axis of [outer][n][inner] fp64
// arrays, N = n + 1 a power of two (4 .. 8192).
//
// Algorithm (per tile of C = 2*NFFT lines, all in shared memory):
//   1. load + pre-process (fused): y_j = s_j (x_j + x_{N-j}) + (x_j - x_{N-j})/2,
//      y_{N-j} = s_j (x_j + x_{N-j}) - (x_j - x_{N-j})/2, s_j = sin(pi j / N),
//      y_0 = 0, y_{N/2} = 2 x_{N/2}.  Lines 2p and 2p+1 become the real and
//      imaginary parts of complex sequence p (two real FFTs for one complex FFT).
//   2. complex DIF FFT of length N in place, radix-8 stages (+ one radix-2/4);
//      frequency k ends up in cell perm(k) (digit reversal, computed inline).
//   3. post-process in place: Y^a_k = (C_k + conj C_{N-k})/2,
//      Y^b_k = (C_k - conj C_{N-k})/(2i); the even output S_{2k} = -Im Y_k goes
//      to cell perm(k), Re Y_k to cell perm(N-k); a segmented scan over k then
//      turns Re Y into the odd outputs S_{2k+1} = Re Y_0/2 + sum_{m<=k} Re Y_m.
//   4. store row j from its cell (even rows from perm(j/2), odd rows from
//      perm(N - (j-1)/2)); the fused operator pass instead scales by the core
//      tensor and runs steps 1-3 again before storing.
// Shared-memory layout: complex cells [pos][p], p (FFT index in the tile)
// fastest.  Contiguous-line tiles (which are transposed on load) XOR-swizzle
// p by key(pos) = low chunk of pos ^ the chunk holding k's low digit after
// digit reversal; the key is XOR-linear, so a cell address assembled from
// disjoint bit fields needs one XOR with a compile-time constant.
// Global access: items are cell columns (line pairs 2p, 2p+1); on strided
// tiles with 16-byte aligned pairs each item is one 16-byte load/store.
// The fused pass reads the DIT input through a shared-memory gather table.
#pragma once

#include "common.cuh"

namespace fl {

// LOAD_PLAIN_TW3: plain loads, DIF twiddles as 3 table loads + products
// (cheaper on the LSU pipe; pays off when the tile accesses are scalar)
enum { LOAD_PLAIN = 0, LOAD_KR = 1, LOAD_PLAIN_TW3 = 2 };

// n / d for 0 <= n < 2^31 without a division: q = (umulhi(n, m) + n) >> s
// with s = ceil(log2 d), m = floor(2^32 (2^s - d) / d) + 1 (set on the host)
struct FastDiv {
  uint32_t d, m, s;
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> s; }
};

inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t s = 0;
  while ((1ull << s) < d) ++s;
  FastDiv f;
  f.d = d;
  f.s = s;
  f.m = (uint32_t)((((1ull << s) - d) << 32) / d + 1);
  return f;
}

struct DstArgs {
  const double* x;
  double* y;
  int64_t outer, n;  // contiguous: number of lines; strided: outer blocks
  // strided tiles: column groups of `wv` valid columns (C-column chunks);
  // element (row j, column c of group g, block o) at o*os + g*gp + c + j*js.
  // contiguous tiles: line L, row j at L*lp + j.  in_* address x (and the
  // core), out_* address y: a pass can change the layout (e.g. pad rows).
  int64_t groups, wv;
  int64_t in_os, in_js, in_gp, in_lp;
  int64_t out_os, out_js, out_gp, out_lp;
  int64_t ntiles, nchunks;
  FastDiv div_blk, div_chunk;  // strided tiles: by groups*nchunks and by nchunks
  // strided tiles: line pairs (2u, 2u+1) are 16-byte aligned on this side
  // (even strides and offsets, 16-byte aligned base and core): one vector
  // access per pair
  int vec_in, vec_out;
  // contiguous output into an internal padded buffer (pitch > n): write
  // zeros into the padding position, so that later passes that pair the
  // last line/column with the padding see a defined value
  int pad_zero;
  double scale;             // applied at the final store
  const double* core;       // fused pass: core tensor, same layout as x
  // LOAD_KR: virtual input Z[j][c] = U[j][c / S] * Xs[j][c % S], wv = R*S
  const double* U;
  const double* Xs;
  int64_t R, S;
  // per-N tables
  const double2* tw;  // N twiddles exp(-2 pi i m / N)
  const double* sn;   // N/2 + 1 values sin(pi j / N)
};

template <int LOGN>
struct FftPlan {
  static constexpr int N = 1 << LOGN;
  static constexpr int NST = (LOGN + 2) / 3;
  static constexpr int rlog(int s) { return s < LOGN / 3 ? 3 : LOGN % 3; }
};

// cell holding frequency k after the DIF stages (digit reversal of k)
template <int LOGN>
__device__ __forceinline__ int perm_of(int k) {
  using P = FftPlan<LOGN>;
  int pos = 0, lg = LOGN;
#pragma unroll
  for (int s = 0; s < P::NST; ++s) {
    const int rl = P::rlog(s);
    lg -= rl;
    pos |= (k & ((1 << rl) - 1)) << lg;
    k >>= rl;
  }
  return pos;
}

template <int LOGN, int LOGF, bool SWZ>
__host__ __device__ constexpr int swz_key(int pos) {
  if (!SWZ || LOGF == 0) return 0;
  // low chunk XOR the chunk where the digit reversal puts k's low digit:
  // a window of consecutive natural positions (load phase) and a window of
  // consecutive k in digit-reversed positions (post/store phases) both see
  // distinct keys, except where a window straddles a chunk boundary
  constexpr int S = LOGN - FftPlan<LOGN>::rlog(0);
  if (S >= LOGF) return (pos ^ (pos >> S)) & ((1 << LOGF) - 1);
  int k = 0;
  for (int sh = 0; sh < LOGN; sh += LOGF) k ^= (pos >> sh);
  return k & ((1 << LOGF) - 1);
}

template <int LOGN, int NFFT, bool SWZ>
struct Cells {
  static constexpr int LOGF = NFFT == 1 ? 0 : NFFT == 2 ? 1 : NFFT == 4 ? 2 : NFFT == 8 ? 3 : 4;
  double2* D;
  __device__ __forceinline__ static int idx(int pos, int p) {
    return pos * NFFT + (p ^ swz_key<LOGN, LOGF, SWZ>(pos));
  }
  // swizzle key of a position; XOR-linear in pos, so the key of a position
  // assembled from disjoint bit fields is the XOR of the fields' keys
  __host__ __device__ static constexpr int key(int pos) { return swz_key<LOGN, LOGF, SWZ>(pos); }
  __device__ __forceinline__ static int idx_k(int pos, int k, int p) { return pos * NFFT + (p ^ k); }
  __device__ __forceinline__ double2 ld(int pos, int p) const { return D[idx(pos, p)]; }
  __device__ __forceinline__ void st(int pos, int p, double2 v) const { D[idx(pos, p)] = v; }
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
  dft4(a[0], a[2], a[4], a[6]);
  dft4(a[1], a[3], a[5], a[7]);
  double2 o1 = a[3], o2 = a[5], o3 = a[7];
  o1 = make_double2((o1.x + o1.y) * r, (o1.y - o1.x) * r);   // * (1 - i)/sqrt2
  o2 = cmul_mi(o2);                                          // * -i
  o3 = make_double2((o3.y - o3.x) * r, -(o3.x + o3.y) * r);  // * (-1 - i)/sqrt2
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

// one DIF stage: sub-length L = 2^LGL, radix R = 2^RL, stride st = L / R.
// Point t of butterfly (block, j) sits at base | (t << LGST): the bits of
// base and t*ST are disjoint, so the swizzle key splits into key(base) ^ K(t).
template <int LOGN, int NFFT, int NT, bool SWZ, int LGL, int RL, bool TW3>
__device__ __forceinline__ void fft_stage(const Cells<LOGN, NFFT, SWZ>& cs, const double2* __restrict__ tw) {
  using CS = Cells<LOGN, NFFT, SWZ>;
  constexpr int N = 1 << LOGN;
  constexpr int R = 1 << RL;
  constexpr int LGST = LGL - RL;
  constexpr int ST = 1 << LGST;
  constexpr int NB = NFFT * (N / R);
  constexpr int PER = (NB + NT - 1) / NT;
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int b = threadIdx.x + it * NT;
    if (NB % NT == 0 || b < NB) {
      const int p = b % NFFT;
      const int bi = b / NFFT;
      const int j = bi & (ST - 1);
      const int base = ((bi >> LGST) << LGL) + j;
      const int pk = p ^ swz_key<LOGN, CS::LOGF, SWZ>(base);
      double2* row = cs.D + base * NFFT;
      double2 v[R];
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = row[t * ST * NFFT + (pk ^ swz_key<LOGN, CS::LOGF, SWZ>(t << LGST))];
      dftR<RL>(v);
      if constexpr (LGST > 0 && !TW3) {
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmul(v[q], __ldg(&tw[(j * q) << (LOGN - LGL)]));
      }
      if constexpr (LGST > 0 && TW3) {
        // twiddles W^{jq}: W^j, W^2j, W^4j from the table, the rest as products
        constexpr int SH = LOGN - LGL;
        const double2 w1 = __ldg(&tw[j << SH]);
        v[1] = cmul(v[1], w1);
        if constexpr (R >= 4) {
          const double2 w2 = __ldg(&tw[(2 * j) << SH]);
          const double2 w3 = cmul(w1, w2);
          v[2] = cmul(v[2], w2);
          v[3] = cmul(v[3], w3);
          if constexpr (R == 8) {
            const double2 w4 = __ldg(&tw[(4 * j) << SH]);
            v[4] = cmul(v[4], w4);
            v[5] = cmul(v[5], cmul(w1, w4));
            v[6] = cmul(v[6], cmul(w2, w4));
            v[7] = cmul(v[7], cmul(w3, w4));
          }
        }
      }
#pragma unroll
      for (int q = 0; q < R; ++q) row[q * ST * NFFT + (pk ^ swz_key<LOGN, CS::LOGF, SWZ>(q << LGST))] = v[q];
    }
  }
  __syncthreads();
}

template <int LOGN, int NFFT, int NT, bool SWZ, int S, int LGL, bool TW3 = false>
__device__ __forceinline__ void fft_rec(const Cells<LOGN, NFFT, SWZ>& cs, const double2* __restrict__ tw) {
  if constexpr (S < FftPlan<LOGN>::NST) {
    constexpr int RL = FftPlan<LOGN>::rlog(S);
    fft_stage<LOGN, NFFT, NT, SWZ, LGL, RL, TW3>(cs, tw);
    fft_rec<LOGN, NFFT, NT, SWZ, S + 1, LGL - RL, TW3>(cs, tw);
  }
}

// frequency held by cell c after the DIF stages (inverse digit reversal)
template <int LOGN>
__device__ __forceinline__ int perm_inv(int c) {
  using P = FftPlan<LOGN>;
  int k = 0, lg = LOGN, sh = 0;
#pragma unroll
  for (int s = 0; s < P::NST; ++s) {
    const int rl = P::rlog(s);
    lg -= rl;
    k |= ((c >> lg) & ((1 << rl) - 1)) << sh;
    sh += rl;
  }
  return k;
}

// DIT stage = transpose of the DIF stage with the same (LGL, RL): twiddles
// before the butterfly.  Running the DIF stages transposed in reverse order
// maps digit-reversed input (cell perm(j) holds x_j) to natural-order output.
template <int LOGN, int NFFT, int NT, bool SWZ, int LGL, int RL>
__device__ __forceinline__ void dit_stage(const Cells<LOGN, NFFT, SWZ>& cs, const double2* __restrict__ tw) {
  using CS = Cells<LOGN, NFFT, SWZ>;
  constexpr int N = 1 << LOGN;
  constexpr int R = 1 << RL;
  constexpr int LGST = LGL - RL;
  constexpr int ST = 1 << LGST;
  constexpr int NB = NFFT * (N / R);
  constexpr int PER = (NB + NT - 1) / NT;
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int b = threadIdx.x + it * NT;
    if (NB % NT == 0 || b < NB) {
      const int p = b % NFFT;
      const int bi = b / NFFT;
      const int j = bi & (ST - 1);
      const int base = ((bi >> LGST) << LGL) + j;
      const int pk = p ^ swz_key<LOGN, CS::LOGF, SWZ>(base);
      double2* row = cs.D + base * NFFT;
      double2 v[R];
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = row[t * ST * NFFT + (pk ^ swz_key<LOGN, CS::LOGF, SWZ>(t << LGST))];
      if constexpr (LGST > 0) {
        // twiddles before the butterfly: W^j, W^2j, W^4j from the table, the
        // rest as products (7 table loads in flight next to R points spill)
        constexpr int SH = LOGN - LGL;
        const double2 w1 = __ldg(&tw[j << SH]);
        v[1] = cmul(v[1], w1);
        if constexpr (R >= 4) {
          const double2 w2 = __ldg(&tw[(2 * j) << SH]);
          v[2] = cmul(v[2], w2);
          const double2 w3 = cmul(w1, w2);
          v[3] = cmul(v[3], w3);
          if constexpr (R == 8) {
            const double2 w4 = __ldg(&tw[(4 * j) << SH]);
            v[4] = cmul(v[4], w4);
            v[5] = cmul(v[5], cmul(w1, w4));
            v[6] = cmul(v[6], cmul(w2, w4));
            v[7] = cmul(v[7], cmul(w3, w4));
          }
        }
      }
      dftR<RL>(v);
#pragma unroll
      for (int q = 0; q < R; ++q) row[q * ST * NFFT + (pk ^ swz_key<LOGN, CS::LOGF, SWZ>(q << LGST))] = v[q];
    }
  }
  __syncthreads();
}

// DIF stage index S -> log2 of its sub-length
template <int LOGN, int S>
struct StageLGL {
  static constexpr int value = S == 0 ? LOGN : StageLGL<LOGN, (S > 0 ? S - 1 : 0)>::value - FftPlan<LOGN>::rlog(S - 1);
};
template <int LOGN>
struct StageLGL<LOGN, 0> {
  static constexpr int value = LOGN;
};

// DIT stages for DIF stages S, S-1, ..., 0
template <int LOGN, int NFFT, int NT, bool SWZ, int S>
__device__ __forceinline__ void dit_rec(const Cells<LOGN, NFFT, SWZ>& cs, const double2* __restrict__ tw) {
  if constexpr (S >= 0) {
    dit_stage<LOGN, NFFT, NT, SWZ, StageLGL<LOGN, S>::value, FftPlan<LOGN>::rlog(S)>(cs, tw);
    dit_rec<LOGN, NFFT, NT, SWZ, S - 1>(cs, tw);
  }
}

// post-process geometry: thread t -> FFT p = t % NFFT, rank g = t / NFFT,
// rank g owns frequencies [g*KPT, (g+1)*KPT)
template <int LOGN, int NFFT, int NT>
struct PostShape {
  static constexpr int H = (1 << LOGN) / 2;
  static constexpr int G0 = NT / NFFT;
  static constexpr int G = G0 < H ? G0 : H;
  static constexpr int KPT = H / G;
  static constexpr int NW = NT / 32;
};

// exclusive scan over ranks g (threads with equal p, stride NFFT)
template <int LOGN, int NFFT, int NT>
__device__ __forceinline__ double2 rank_excl_scan(double2 v, double2* scr) {
  using PS = PostShape<LOGN, NFFT, NT>;
  const int lane = threadIdx.x & 31;
  const int warp = threadIdx.x >> 5;
  double2 x = v;
  if constexpr (NFFT < 32) {
#pragma unroll
    for (int d = NFFT; d < 32; d <<= 1) {
      const double yx = __shfl_up_sync(0xffffffffu, x.x, d);
      const double yy = __shfl_up_sync(0xffffffffu, x.y, d);
      if (lane >= d) {
        x.x += yx;
        x.y += yy;
      }
    }
  }
  if constexpr (PS::NW == 1) {
    return make_double2(x.x - v.x, x.y - v.y);
  } else {
    // warp totals per p live in the last NFFT lanes
    if (lane >= 32 - NFFT) scr[warp * NFFT + (lane & (NFFT - 1))] = x;
    __syncthreads();
    // warp 0 scans the NW totals of every p in place: lane (p, q) owns a run
    // of WPL consecutive warps, runs are combined with shuffles over q
    if (warp == 0) {
      constexpr int LPP = 32 / NFFT;
      constexpr int WPL = (PS::NW + LPP - 1) / LPP;
      const int p = lane & (NFFT - 1), q = lane / NFFT;
      double2 loc[WPL];
      double2 sum = make_double2(0.0, 0.0);
#pragma unroll
      for (int i = 0; i < WPL; ++i) {
        const int w = q * WPL + i;
        loc[i] = (w < PS::NW) ? scr[w * NFFT + p] : make_double2(0.0, 0.0);
        sum.x += loc[i].x;
        sum.y += loc[i].y;
      }
      double2 inc = sum;
#pragma unroll
      for (int d = NFFT; d < 32; d <<= 1) {
        const double yx = __shfl_up_sync(0xffffffffu, inc.x, d);
        const double yy = __shfl_up_sync(0xffffffffu, inc.y, d);
        if (lane >= d) {
          inc.x += yx;
          inc.y += yy;
        }
      }
      double2 run = make_double2(inc.x - sum.x, inc.y - sum.y);
#pragma unroll
      for (int i = 0; i < WPL; ++i) {
        const int w = q * WPL + i;
        if (w < PS::NW) scr[w * NFFT + p] = run;
        run.x += loc[i].x;
        run.y += loc[i].y;
      }
    }
    __syncthreads();
    // scr is next written by the following post-process, after its barriers
    const double2 o = scr[warp * NFFT + (threadIdx.x & (NFFT - 1))];
    return make_double2(x.x - v.x + o.x, x.y - v.y + o.y);
  }
}

// compile-time digit reversal (host/device constexpr twin of perm_of)
template <int LOGN>
__host__ __device__ constexpr int perm_c(int k) {
  int pos = 0, lg = LOGN;
  for (int s = 0; s < FftPlan<LOGN>::NST; ++s) {
    const int rl = FftPlan<LOGN>::rlog(s);
    lg -= rl;
    pos |= (k & ((1 << rl) - 1)) << lg;
    k >>= rl;
  }
  return pos;
}

// Cells of frequency k and N-k for k = k0 + m*S (S a power of two, k0 < S):
// digit reversal acts on disjoint bit fields, so perm(k) = perm(k0) | perm(m*S)
// and, with N - k = ~(k - 1), perm(N - k) = (N-1) - (perm(k0-1) | perm(m*S)).
struct KCells {
  int pe;   // perm(k0)
  int po;   // (N-1) - perm(k0-1) = (N-1) ^ perm(k0-1), unused when k0 == 0
  bool z;   // k0 == 0
  int ke, ko;  // swizzle keys of pe and po
};

// NAT: natural order (cell k holds frequency k), the layout after DIT stages
template <int LOGN, class CS, bool NAT = false>
__device__ __forceinline__ KCells kcells(int k0) {
  KCells c;
  c.pe = NAT ? k0 : perm_of<LOGN>(k0);
  c.z = (k0 == 0);
  c.po = (1 << LOGN) - 1 - (NAT ? k0 - 1 : perm_of<LOGN>(k0 - 1));
  c.ke = CS::key(c.pe);
  c.ko = CS::key(c.po);
  return c;
}

// ms is a compile-time constant after loop unrolling; perm_c folds away
template <int LOGN, bool NAT = false>
__device__ __forceinline__ int cell_even(const KCells& c, int ms) {
  return c.pe | (NAT ? ms : perm_c<LOGN>(ms));
}

template <int LOGN, bool NAT = false>
__device__ __forceinline__ int cell_odd(const KCells& c, int ms) {
  constexpr int N = 1 << LOGN;
  const int zp = (N - ms) & (N - 1);
  return c.z ? (NAT ? zp : perm_c<LOGN>(zp)) : c.po ^ (NAT ? ms : perm_c<LOGN>(ms));
}

// cell indices of the two cells above with the swizzle key assembled from
// the per-thread keys and compile-time parts
template <int LOGN, class CS, bool NAT = false>
__device__ __forceinline__ int even_idx(const KCells& c, int ms, int p) {
  const int b = NAT ? ms : perm_c<LOGN>(ms);
  return CS::idx_k(c.pe | b, c.ke ^ CS::key(b), p);
}

template <int LOGN, class CS, bool NAT = false>
__device__ __forceinline__ int odd_idx(const KCells& c, int ms, int p) {
  constexpr int N = 1 << LOGN;
  const int zp = (N - ms) & (N - 1);
  const int b = NAT ? ms : perm_c<LOGN>(ms);
  return c.z ? CS::idx(NAT ? zp : perm_c<LOGN>(zp), p) : CS::idx_k(c.po ^ b, c.ko ^ CS::key(b), p);
}

// in-place post-process (see header); leaves even outputs in perm(k) and odd
// outputs in perm(N-k), unscaled.  Rank g owns k in [g*KPT, (g+1)*KPT), i.e.
// k = i + g*KPT with the roles of (k0, m*S) swapped: perm(k) = perm(i) | A.
template <int LOGN, int NFFT, int NT, bool SWZ, bool NAT = false>
__device__ __forceinline__ void dst_post(const Cells<LOGN, NFFT, SWZ>& cs, double2* scr) {
  using PS = PostShape<LOGN, NFFT, NT>;
  using CS = Cells<LOGN, NFFT, SWZ>;
  constexpr int N = 1 << LOGN;
  constexpr int K = PS::KPT;
  const int p = threadIdx.x % NFFT;
  const int g = threadIdx.x / NFFT;
  const bool active = g < PS::G;
  // NAT: spectrum in natural order (cell k holds frequency k)
  const int A = NAT ? g * K : perm_of<LOGN>(g * K);
  const int B = (g == 0) ? 0 : (NAT ? N - g * K : (N - 1 - perm_of<LOGN>(g * K - 1)));
  // cell indices: A and the compile-time parts are disjoint bit fields, so
  // positions and swizzle keys combine by XOR
  const int kA = CS::key(A), kB = CS::key(B);
  constexpr int KN = CS::key(N - 1);
  auto ck_idx = [&](int i) {
    const int b = NAT ? i : perm_c<LOGN>(i);
    return CS::idx_k(A | b, kA ^ CS::key(b), p);
  };
  auto cm_idx = [&](int i) {
    if (i == 0) return CS::idx_k(B, kB, p);
    const int b = NAT ? i - 1 : perm_c<LOGN>(i - 1);
    return CS::idx_k((N - 1) ^ A ^ b, KN ^ kA ^ CS::key(b), p);
  };
  double2 tot = make_double2(0.0, 0.0);
  // P1: split the packed spectra pairwise (k, N-k); R_k summed on the fly
  if (active) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int ik = ck_idx(i), im = cm_idx(i);
      const double2 ck = cs.D[ik];
      const double2 cm = cs.D[im];
      const double2 e = make_double2(0.5 * (cm.y - ck.y), 0.5 * (ck.x - cm.x));
      double2 r = make_double2(0.5 * (ck.x + cm.x), 0.5 * (ck.y + cm.y));
      if (i == 0 && g == 0) {
        r.x *= 0.5;
        r.y *= 0.5;
        cs.D[ik] = r;  // cell 0 seeds S_1; S_0 = 0 is implicit
      } else {
        cs.D[ik] = e;
        cs.D[im] = r;
      }
      tot.x += r.x;
      tot.y += r.y;
    }
  }
  // P2: segmented prefix sum of Re Y over k -> odd outputs
  double2 run = rank_excl_scan<LOGN, NFFT, NT>(tot, scr);
  if (active) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int im = cm_idx(i);
      const double2 r = cs.D[im];
      run.x += r.x;
      run.y += r.y;
      cs.D[im] = run;
    }
  }
  __syncthreads();
}

// cell position of natural output row j after dst_post (j in [1, N-1])
template <int LOGN>
__device__ __forceinline__ int out_pos(int j) {
  constexpr int N = 1 << LOGN;
  return (j & 1) ? perm_of<LOGN>((N - (j >> 1)) & (N - 1)) : perm_of<LOGN>(j >> 1);
}

template <int LOGN, int NFFT, bool SWZ>
__device__ __forceinline__ double out_elem(const Cells<LOGN, NFFT, SWZ>& cs, int l, int j) {
  return reinterpret_cast<const double*>(cs.D)[2 * Cells<LOGN, NFFT, SWZ>::idx(out_pos<LOGN>(j), l >> 1) + (l & 1)];
}

// Opaque copy: stops the compiler from carrying values (and everything it
// derived from them) across phases, which otherwise blows the register file.
__device__ __forceinline__ int64_t launder(int64_t v) {
  int64_t r;
  asm volatile("mov.b64 %0, %1;" : "=l"(r) : "l"(v));
  return r;
}
__device__ __forceinline__ int launder(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// per-tile addressing: element (l, j) (j in [1, n]) at base + l*LS + (j-1)*JS
struct TileAddr {
  int64_t base;  // element offset of (0, 1)
  int64_t JS;
  int LS;
  int lmax;  // lines [0, lmax) are valid
  int64_t c0;
  __device__ __forceinline__ TileAddr fresh() const {
    TileAddr t;
    t.base = launder(base);
    t.JS = launder(JS);
    t.LS = launder(LS);
    t.lmax = launder(lmax);
    t.c0 = launder(c0);
    return t;
  }
};

template <bool CONTIG, int C, bool OUT = false>
__device__ __forceinline__ TileAddr tile_addr(const DstArgs& a, int64_t tile) {
  TileAddr t;
  if (CONTIG) {
    const int64_t L0 = tile * C;
    const int64_t lp = OUT ? a.out_lp : a.in_lp;
    t.base = L0 * lp;
    t.JS = 1;
    t.LS = (int)lp;
    const int64_t rem = a.outer - L0;
    t.lmax = (int)(rem < C ? rem : C);
    t.c0 = 0;
  } else {
    // tile = (o * groups + g) * nchunks + chunk, ntiles < 2^31
    const uint32_t t32 = (uint32_t)tile;
    const uint32_t o = a.div_blk.div(t32);
    const uint32_t r = t32 - o * a.div_blk.d;
    const uint32_t g = a.div_chunk.div(r);
    const int64_t c0 = (int64_t)(r - g * a.div_chunk.d) * C;
    t.base = (int64_t)o * (OUT ? a.out_os : a.in_os) + (int64_t)g * (OUT ? a.out_gp : a.in_gp) + c0;
    t.JS = OUT ? a.out_js : a.in_js;
    t.LS = 1;
    const int64_t rem = a.wv - c0;
    t.lmax = (int)(rem < C ? rem : C);
    t.c0 = c0;
  }
  return t;
}

// Work split shared by the load, fused-core and store phases: items (u, k),
// u a cell column (tile lines 2u and 2u+1, the re/im halves of one packed
// FFT) and k in [0, H) a row pair; NFFT*H items over NT threads, PER each.
// Strided tiles: u = t % NFFT fixed, k = t / NFFT + it * (NT / NFFT), so a
// warp access covers 32/NFFT rows of 2*NFFT consecutive columns.
// Contiguous tiles: k = t % H (+ multiples of NT when NT < H), u varies.
template <int LOGN, int NFFT, int NT, bool CONTIG>
struct Split {
  static constexpr int N = 1 << LOGN;
  static constexpr int H = N / 2;
  static constexpr int ITEMS = NFFT * H;
  static constexpr int PER = (ITEMS + NT - 1) / NT;
  // k = k0 + MS(it), u = u0 + LD(it)
  __device__ __forceinline__ static void base(int t, int& k0, int& u0) {
    if (CONTIG) {
      k0 = (NT >= H) ? (t % H) : t;
      u0 = (NT >= H) ? (t / H) : 0;
    } else {
      k0 = t / NFFT;
      u0 = t % NFFT;
    }
  }
  __host__ __device__ static constexpr int MS(int it) {
    return CONTIG ? ((NT >= H) ? 0 : (it % (H / NT)) * NT) : it * (NT / NFFT);
  }
  __host__ __device__ static constexpr int LD(int it) {
    return CONTIG ? ((NT >= H) ? it * (NT / H) : it / (H / NT)) : 0;
  }
  __device__ __forceinline__ static bool ok(int t, int it) { return ITEMS % NT == 0 || t + it * NT < ITEMS; }
};

template <int LOADER>
__device__ __forceinline__ double load_elem(const DstArgs& a, const TileAddr& ta, int l, int row) {
  if constexpr (LOADER != LOAD_KR) {
    return __ldg(&a.x[ta.base + (int64_t)l * ta.LS + (int64_t)row * ta.JS]);
  } else {
    const int64_t c = ta.c0 + l;
    const int64_t k = c / a.S, s = c - k * a.S;
    return __ldg(&a.U[(int64_t)row * a.R + k]) * __ldg(&a.Xs[(int64_t)row * a.S + s]);
  }
}

// the pair (lines 2u, 2u+1) at element pointer p: one 16-byte access when
// the layout keeps pairs aligned (VEC), else two (line 2u+1 may be absent)
__device__ __forceinline__ double2 ld_pair(const double* p, int64_t ls, bool vec, bool hi) {
  if (vec) return __ldg(reinterpret_cast<const double2*>(p));
  return make_double2(__ldg(p), hi ? __ldg(p + ls) : 0.0);
}

__device__ __forceinline__ void st_pair(double* p, int64_t ls, bool vec, bool hi, double2 v) {
  if (vec) {
    *reinterpret_cast<double2*>(p) = v;
  } else {
    p[0] = v.x;
    if (hi) p[ls] = v.y;
  }
}

// DST-I pre-processing of rows (j, N-j) of cell column u from pairs (va, vb)
template <int LOGN, int NFFT, bool SWZ>
__device__ __forceinline__ void pre_pair(const Cells<LOGN, NFFT, SWZ>& cs, const double* __restrict__ sn, int u, int j,
                                         double2 va, double2 vb) {
  constexpr int H = (1 << LOGN) / 2;
  if (j == H) {
    cs.st(H, u, make_double2(2.0 * va.x, 2.0 * va.y));
  } else {
    const double s = __ldg(&sn[j]);
    const double sx = s * (va.x + vb.x), dx = 0.5 * (va.x - vb.x);
    const double sy = s * (va.y + vb.y), dy = 0.5 * (va.y - vb.y);
    cs.st(j, u, make_double2(sx + dx, sy + dy));
    cs.st((1 << LOGN) - j, u, make_double2(sx - dx, sy - dy));
  }
}

// stage 1: global -> smem with the DST-I pre-processing fused in.  Item
// (u, k) covers rows j = k + 1 and N - j of lines 2u, 2u+1.  A batch of a
// thread's loads is issued before any is consumed; addresses advance by
// per-item constant strides.
template <int LOGN, int NFFT, int NT, bool CONTIG, int LOADER>
__device__ __forceinline__ void dst_load_pre(const DstArgs& a, const Cells<LOGN, NFFT, CONTIG>& cs,
                                             const TileAddr& ta) {
  using SP = Split<LOGN, NFFT, NT, CONTIG>;
  constexpr int N = SP::N, H = SP::H, PER = SP::PER;
  constexpr int B = PER < 4 ? PER : 4;
  static_assert(PER % B == 0, "batch must divide the per-thread item count");
  int k0, u0;
  SP::base(threadIdx.x, k0, u0);
  if constexpr (LOADER != LOAD_KR) {
    const bool vec = !CONTIG && a.vec_in;
    const int64_t LS = ta.LS;
    const double* xp = a.x + ta.base + (int64_t)(2 * u0) * LS;
    const double* pa = xp + (int64_t)k0 * ta.JS;            // row j - 1 = k
    const double* pb = xp + (int64_t)(N - 2 - k0) * ta.JS;  // row N - j - 1
#pragma unroll
    for (int it0 = 0; it0 < PER; it0 += B) {
      double2 xa[B], xb[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int it = it0 + u;
        const int l = 2 * (u0 + SP::LD(it));
        const int k = k0 + SP::MS(it);
        const int64_t lo = (int64_t)(2 * SP::LD(it)) * LS;
        xa[u] = make_double2(0.0, 0.0);
        xb[u] = make_double2(0.0, 0.0);
        if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
          const bool hi = l + 1 < ta.lmax;
          xa[u] = ld_pair(pa + lo + (int64_t)SP::MS(it) * ta.JS, LS, vec, hi);
          if (k + 1 < H) xb[u] = ld_pair(pb + lo - (int64_t)SP::MS(it) * ta.JS, LS, vec, hi);
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int it = it0 + u;
        if (SP::ok(threadIdx.x, it)) pre_pair(cs, a.sn, u0 + SP::LD(it), k0 + SP::MS(it) + 1, xa[u], xb[u]);
      }
    }
  } else {
#pragma unroll
    for (int it0 = 0; it0 < PER; it0 += B) {
      double2 xa[B], xb[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int it = it0 + u;
        const int l = 2 * (u0 + SP::LD(it));
        const int j = k0 + SP::MS(it) + 1;
        xa[u] = make_double2(0.0, 0.0);
        xb[u] = make_double2(0.0, 0.0);
        if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
          const bool hi = l + 1 < ta.lmax;
          xa[u].x = load_elem<LOADER>(a, ta, l, j - 1);
          if (hi) xa[u].y = load_elem<LOADER>(a, ta, l + 1, j - 1);
          if (j < H) {
            xb[u].x = load_elem<LOADER>(a, ta, l, N - j - 1);
            if (hi) xb[u].y = load_elem<LOADER>(a, ta, l + 1, N - j - 1);
          }
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int it = it0 + u;
        if (SP::ok(threadIdx.x, it)) pre_pair(cs, a.sn, u0 + SP::LD(it), k0 + SP::MS(it) + 1, xa[u], xb[u]);
      }
    }
  }
  for (int u = threadIdx.x; u < NFFT; u += NT) cs.st(0, u, make_double2(0.0, 0.0));
}

// Line-based split (strided tiles whose line pairs are not 16-byte aligned):
// items (l, k),
// k in [0, H) (a row pair), C*H items over NT threads, PER per thread.
// Strided tiles: l = t % C fixed, k = t / C + it * (NT / C).
// Contiguous tiles: k = t % H (+ multiples of NT when NT < H), l varies.
template <int LOGN, int NFFT, int NT, bool CONTIG>
struct SplitL {
  static constexpr int N = 1 << LOGN;
  static constexpr int H = N / 2;
  static constexpr int C = 2 * NFFT;
  static constexpr int ITEMS = C * H;
  static constexpr int PER = (ITEMS + NT - 1) / NT;
  // k = k0 + MS(it), l = l0 + LD(it)
  __device__ __forceinline__ static void base(int t, int& k0, int& l0) {
    if (CONTIG) {
      k0 = (NT >= H) ? (t % H) : t;
      l0 = (NT >= H) ? (t / H) : 0;
    } else {
      k0 = t / C;
      l0 = t % C;
    }
  }
  __host__ __device__ static constexpr int MS(int it) {
    return CONTIG ? ((NT >= H) ? 0 : (it % (H / NT)) * NT) : it * (NT / C);
  }
  __host__ __device__ static constexpr int LD(int it) {
    return CONTIG ? ((NT >= H) ? it * (NT / H) : it / (H / NT)) : 0;
  }
  __host__ __device__ static constexpr int KS() {  // S of the k = k0 + m*S form
    return CONTIG ? ((NT >= H) ? H : NT) : (NT / C);
  }
  __device__ __forceinline__ static bool ok(int t, int it) { return ITEMS % NT == 0 || t + it * NT < ITEMS; }
};

// DST-I pre-processing of rows (j, N-j) of one line l from values (va, vb)
template <int LOGN, int NFFT, bool SWZ>
__device__ __forceinline__ void pre_line(const Cells<LOGN, NFFT, SWZ>& cs, const double* __restrict__ sn, int l, int j,
                                         double va, double vb) {
  constexpr int H = (1 << LOGN) / 2;
  if (j == H) {
    cs.re(l, H) = 2.0 * va;
  } else {
    const double s = __ldg(&sn[j]);
    const double sum = s * (va + vb), dif = 0.5 * (va - vb);
    cs.re(l, j) = sum + dif;
    cs.re(l, (1 << LOGN) - j) = sum - dif;
  }
}

// stage 1 for strided tiles without aligned line pairs: one item per line;
// item (l, k) covers rows j = k + 1 and N - j.  All of a thread's loads are issued
// before any is consumed; addresses advance by per-item constant strides.
template <int LOGN, int NFFT, int NT>
__device__ __forceinline__ void dst_load_lines(const DstArgs& a, const Cells<LOGN, NFFT, false>& cs,
                                               const TileAddr& ta) {
  using SP = SplitL<LOGN, NFFT, NT, false>;
  constexpr int N = SP::N, H = SP::H, PER = SP::PER;
  constexpr int B = PER < 8 ? PER : 8;
  static_assert(PER % B == 0, "batch must divide the per-thread item count");
  int k0, l0;
  SP::base(threadIdx.x, k0, l0);
  {
    const double* xp = a.x + ta.base + (int64_t)l0 * ta.LS;
    const double* pa = xp + (int64_t)k0 * ta.JS;           // row j - 1 = k
    const double* pb = xp + (int64_t)(N - 2 - k0) * ta.JS; // row N - j - 1
#pragma unroll
    for (int it0 = 0; it0 < PER; it0 += B) {
      double xa[B], xb[B];
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int it = it0 + u;
        const int l = l0 + SP::LD(it);
        const int k = k0 + SP::MS(it);
        const int64_t off = (int64_t)SP::LD(it) * ta.LS + (int64_t)SP::MS(it) * ta.JS;
        xa[u] = 0.0;
        xb[u] = 0.0;
        if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
          xa[u] = __ldg(pa + off);
          if (k + 1 < H) xb[u] = __ldg(pb + (int64_t)SP::LD(it) * ta.LS - (int64_t)SP::MS(it) * ta.JS);
        }
      }
#pragma unroll
      for (int u = 0; u < B; ++u) {
        const int it = it0 + u;
        if (SP::ok(threadIdx.x, it)) pre_line(cs, a.sn, l0 + SP::LD(it), k0 + SP::MS(it) + 1, xa[u], xb[u]);
      }
    }
  }
  for (int l = threadIdx.x; l < SP::C; l += NT) cs.re(l, 0) = 0.0;
}

// value of natural row j (1 <= j <= N-1) of line l after dst_post
template <int LOGN, int NFFT, bool SWZ>
__device__ __forceinline__ double post_val(const Cells<LOGN, NFFT, SWZ>& cs, int l, int cell) {
  return reinterpret_cast<const double*>(cs.D)[2 * Cells<LOGN, NFFT, SWZ>::idx(cell, l >> 1) + (l & 1)];
}

// fused operator pass, step 1: scale the post-processed forward transform by
// the core in place (cells perm(k) / perm(N-k) hold rows 2k / 2k+1), with the
// store's item mapping for the core loads.  Cells are private to the
// thread, so no barrier is needed; items go in register batches of 4.
template <int LOGN, int NFFT, int NT, bool CONTIG>
__device__ __forceinline__ void dst_core_scale(const DstArgs& a, const Cells<LOGN, NFFT, CONTIG>& cs,
                                               const TileAddr& ta_in) {
  const TileAddr ta = ta_in.fresh();
  using SP = Split<LOGN, NFFT, NT, CONTIG>;
  constexpr int PER = SP::PER;
  constexpr int B = PER < 4 ? PER : 4;
  static_assert(PER % B == 0, "batch must divide the per-thread item count");
  int k0, u0;
  SP::base(threadIdx.x, k0, u0);
  const KCells kc = kcells<LOGN, Cells<LOGN, NFFT, CONTIG>>(k0);
  const bool vec = !CONTIG && a.vec_in;
  const int64_t LS = ta.LS;
  const double* cb = a.core + ta.base + (int64_t)(2 * u0) * LS;
#pragma unroll
  for (int it0 = 0; it0 < PER; it0 += B) {
    double2 ce_v[B], co_v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int it = it0 + u;
      const int l = 2 * (u0 + SP::LD(it));
      const int k = k0 + SP::MS(it);
      ce_v[u] = make_double2(0.0, 0.0);
      co_v[u] = make_double2(0.0, 0.0);
      if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
        const bool hi = l + 1 < ta.lmax;
        const double* cl = cb + (int64_t)(2 * SP::LD(it)) * LS;
        co_v[u] = ld_pair(cl + (int64_t)(2 * k) * ta.JS, LS, vec, hi);
        if (k > 0) ce_v[u] = ld_pair(cl + (int64_t)(2 * k - 1) * ta.JS, LS, vec, hi);
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int it = it0 + u;
      const int p = u0 + SP::LD(it);
      if (SP::ok(threadIdx.x, it)) {
        using CS = Cells<LOGN, NFFT, CONTIG>;
        const int io = odd_idx<LOGN, CS>(kc, SP::MS(it), p);
        const double2 vo = cs.D[io];
        cs.D[io] = make_double2(vo.x * co_v[u].x, vo.y * co_v[u].y);
        if (k0 + SP::MS(it) > 0) {
          const int ie = even_idx<LOGN, CS>(kc, SP::MS(it), p);
          const double2 ve = cs.D[ie];
          cs.D[ie] = make_double2(ve.x * ce_v[u].x, ve.y * ce_v[u].y);
        }
      }
    }
  }
}

// Gather table of the fused pass (N <= 1024): entry for DIT-input cell c =
// the two source cells of y_j, j = perm_inv(c) (rows j and N - j), packed
// as (pos * NFFT) << 4 | swizzle key, and sin(pi j / N) (0 for j = 0, so
// that cell gets 0).  Stored t-major (c % R, c / R) so that the lanes of a
// warp, which share c / R in groups of NFFT, read adjacent entries.
struct __align__(16) GatherEnt {
  int ia, ib;
  double s;
};

template <int LOGN>
struct GatherTable {
  static constexpr bool ON = LOGN <= 10;
  static constexpr size_t bytes() { return ON ? sizeof(GatherEnt) * (size_t(1) << LOGN) : 0; }
};

template <int LOGN, int NFFT, int NT, bool SWZ>
__device__ __forceinline__ void gather_table_fill(const double* __restrict__ sn, GatherEnt* gt) {
  using CS = Cells<LOGN, NFFT, SWZ>;
  constexpr int N = 1 << LOGN;
  constexpr int H = N / 2;
  constexpr int R = 1 << FftPlan<LOGN>::rlog(FftPlan<LOGN>::NST - 1);
  for (int c = threadIdx.x; c < N; c += NT) {
    const int j = perm_inv<LOGN>(c);
    GatherEnt e;
    if (j == 0) {
      e.ia = e.ib = 0;
      e.s = 0.0;
    } else {
      const int pa = out_pos<LOGN>(j);
      const int pb = (j == H) ? pa : out_pos<LOGN>(N - j);
      e.ia = ((pa * NFFT) << 4) | CS::key(pa);
      e.ib = ((pb * NFFT) << 4) | CS::key(pb);
      e.s = sn[j < H ? j : N - j];
    }
    gt[(c % R) * (N / R) + c / R] = e;
  }
}

// fused operator pass, step 2: first DIT stage (transpose of the last DIF
// stage: sub-length R, unit stride, no twiddles) whose inputs are gathered
// from the core-scaled spectrum with the DST-I pre-processing applied on the
// fly.  Cell c of the DIT input holds y_j, j = perm_inv(c); y_j needs rows
// j and N - j, which sit in cells out_pos(j) and out_pos(N - j).  All reads
// finish before the barrier; each thread then writes its own butterfly.
template <int LOGN, int NFFT, int NT, bool CONTIG>
__device__ __forceinline__ void dit_gather_stage(const DstArgs& a, const Cells<LOGN, NFFT, CONTIG>& cs,
                                                 const GatherEnt* __restrict__ gt) {
  using CS = Cells<LOGN, NFFT, CONTIG>;
  constexpr int N = 1 << LOGN;
  constexpr int H = N / 2;
  constexpr int RL = FftPlan<LOGN>::rlog(FftPlan<LOGN>::NST - 1);
  constexpr int R = 1 << RL;
  constexpr int NB = NFFT * (N / R);
  constexpr int PER = (NB + NT - 1) / NT;
  double2 v[PER][R];
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int b = threadIdx.x + it * NT;
    if (NB % NT == 0 || b < NB) {
      const int p = b % NFFT;
      const int base = (b / NFFT) * R;
      if constexpr (GatherTable<LOGN>::ON) {
        const GatherEnt* e = gt + base / R;
#pragma unroll
        for (int t = 0; t < R; ++t) {
          const GatherEnt g = e[t * (N / R)];
          const double2 xa = cs.D[(g.ia >> 4) + ((g.ia & 15) ^ p)];
          const double2 xb = cs.D[(g.ib >> 4) + ((g.ib & 15) ^ p)];
          v[it][t] = make_double2(fma(g.s, xa.x + xb.x, 0.5 * (xa.x - xb.x)), fma(g.s, xa.y + xb.y, 0.5 * (xa.y - xb.y)));
        }
        dftR<RL>(v[it]);
        continue;
      }
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = perm_inv<LOGN>(base + t);
        // y_j = s_j (x_j + x_{N-j}) + (x_j - x_{N-j})/2 holds for every j in [1, N)
        double2 y = make_double2(0.0, 0.0);
        if (j != 0) {
          const double2 xa = cs.ld(out_pos<LOGN>(j), p);
          const double2 xb = (j == H) ? xa : cs.ld(out_pos<LOGN>(N - j), p);
          const double s = __ldg(&a.sn[j < H ? j : N - j]);
          y = make_double2(fma(s, xa.x + xb.x, 0.5 * (xa.x - xb.x)), fma(s, xa.y + xb.y, 0.5 * (xa.y - xb.y)));
        }
        v[it][t] = y;
      }
      dftR<RL>(v[it]);
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int b = threadIdx.x + it * NT;
    if (NB % NT == 0 || b < NB) {
      const int p = b % NFFT;
      const int base = (b / NFFT) * R;
#pragma unroll
      for (int q = 0; q < R; ++q) cs.st(base + q, p, v[it][q]);
    }
  }
  __syncthreads();
}

// store: item (u, k) writes rows 2k (k >= 1) and 2k+1 of lines 2u, 2u+1 from
// cells perm(k) and perm(N-k), addresses linear in the unrolled item index.
template <int LOGN, int NFFT, int NT, bool CONTIG, bool NAT = false>
__device__ __forceinline__ void dst_store(const DstArgs& a, const Cells<LOGN, NFFT, CONTIG>& cs,
                                          const TileAddr& ta_in) {
  const TileAddr ta = ta_in.fresh();
  using SP = Split<LOGN, NFFT, NT, CONTIG>;
  constexpr int PER = SP::PER;
  const double sc = a.scale;
  int k0, u0;
  SP::base(launder((int)threadIdx.x), k0, u0);
  using CS = Cells<LOGN, NFFT, CONTIG>;
  const KCells kc = kcells<LOGN, CS, NAT>(k0);
  const bool vec = !CONTIG && a.vec_out;
  const int64_t LS = ta.LS;
  double* yb = a.y + ta.base + (int64_t)(2 * u0) * LS;
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int l = 2 * (u0 + SP::LD(it));
    const int k = k0 + SP::MS(it);
    if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
      const bool hi = l + 1 < ta.lmax;
      const int p = u0 + SP::LD(it);
      double* yl = yb + (int64_t)(2 * SP::LD(it)) * LS;
      // row 2k+1 -> offset 2k, row 2k -> offset 2k-1
      const double2 vo = cs.D[odd_idx<LOGN, CS, NAT>(kc, SP::MS(it), p)];
      st_pair(yl + (int64_t)(2 * k) * ta.JS, LS, vec, hi, make_double2(sc * vo.x, sc * vo.y));
      if (k > 0) {
        const double2 ve = cs.D[even_idx<LOGN, CS, NAT>(kc, SP::MS(it), p)];
        st_pair(yl + (int64_t)(2 * k - 1) * ta.JS, LS, vec, hi, make_double2(sc * ve.x, sc * ve.y));
      }
    }
  }
}

// store for strided tiles without aligned line pairs, one item per line:
// item (l, k) writes rows 2k (k >= 1) and 2k+1 from cells perm(k) and
// perm(N-k), addresses linear in the unrolled item index.
template <int LOGN, int NFFT, int NT>
__device__ __forceinline__ void dst_store_lines(const DstArgs& a, const Cells<LOGN, NFFT, false>& cs,
                                                const TileAddr& ta_in) {
  const TileAddr ta = ta_in.fresh();
  using SP = SplitL<LOGN, NFFT, NT, false>;
  constexpr int PER = SP::PER;
  const double sc = a.scale;
  int k0, l0;
  SP::base(launder((int)threadIdx.x), k0, l0);
  const KCells kc = kcells<LOGN, Cells<LOGN, NFFT, false>>(k0);
  double* yb = a.y + ta.base + (int64_t)l0 * ta.LS;
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int l = l0 + SP::LD(it);
    const int k = k0 + SP::MS(it);
    if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
      double* yl = yb + (int64_t)SP::LD(it) * ta.LS;
      const int ce = cell_even<LOGN>(kc, SP::MS(it));
      const int co = cell_odd<LOGN>(kc, SP::MS(it));
      // row 2k+1 -> offset 2k, row 2k -> offset 2k-1
      yl[(int64_t)(2 * k) * ta.JS] = sc * post_val(cs, l, co);
      if (k > 0) yl[(int64_t)(2 * k - 1) * ta.JS] = sc * post_val(cs, l, ce);
    }
  }
}

template <int LOGN, int NFFT, int NT, int MINB, bool CONTIG, int LOADER, bool MIDCORE>
__global__ void __launch_bounds__(NT, MINB) k_dst_fft(const DstArgs a) {
  using CS = Cells<LOGN, NFFT, CONTIG>;
  constexpr int C = 2 * NFFT;
  extern __shared__ __align__(16) double smem_dst[];
  CS cs{reinterpret_cast<double2*>(smem_dst)};
  double2* scr = reinterpret_cast<double2*>(smem_dst + 2 * (1 << LOGN) * NFFT);
  GatherEnt* gt = reinterpret_cast<GatherEnt*>(smem_dst + 2 * (1 << LOGN) * NFFT + 2 * NFFT * (NT / 32));
  if constexpr (MIDCORE && GatherTable<LOGN>::ON) gather_table_fill<LOGN, NFFT, NT, CONTIG>(a.sn, gt);
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    // per-tile addressing is recomputed (from a laundered tile index) in every
    // phase that needs it, so nothing address-like stays live across the FFTs
    if constexpr (!CONTIG && LOADER != LOAD_KR) {
      if (a.vec_in) {
        dst_load_pre<LOGN, NFFT, NT, CONTIG, LOADER>(a, cs, tile_addr<CONTIG, C>(a, tile));
      } else {
        dst_load_lines<LOGN, NFFT, NT>(a, cs, tile_addr<CONTIG, C>(a, tile));
      }
    } else {
      dst_load_pre<LOGN, NFFT, NT, CONTIG, LOADER>(a, cs, tile_addr<CONTIG, C>(a, tile));
    }
    __syncthreads();
    fft_rec<LOGN, NFFT, NT, CONTIG, 0, LOGN, LOADER == LOAD_PLAIN_TW3>(cs, a.tw);
    dst_post<LOGN, NFFT, NT, CONTIG>(cs, scr);
    if constexpr (MIDCORE) {
      dst_core_scale<LOGN, NFFT, NT, CONTIG>(a, cs, tile_addr<CONTIG, C>(a, launder(tile)));
      __syncthreads();
      dit_gather_stage<LOGN, NFFT, NT, CONTIG>(a, cs, gt);
      dit_rec<LOGN, NFFT, NT, CONTIG, FftPlan<LOGN>::NST - 2>(cs, a.tw);
      dst_post<LOGN, NFFT, NT, CONTIG, true>(cs, scr);
      dst_store<LOGN, NFFT, NT, CONTIG, true>(a, cs, tile_addr<CONTIG, C, true>(a, launder(tile)));
    } else {
      if constexpr (!CONTIG) {
        if (a.vec_out) {
          dst_store<LOGN, NFFT, NT, CONTIG>(a, cs, tile_addr<CONTIG, C, true>(a, launder(tile)));
        } else {
          dst_store_lines<LOGN, NFFT, NT>(a, cs, tile_addr<CONTIG, C, true>(a, launder(tile)));
        }
      } else {
        dst_store<LOGN, NFFT, NT, CONTIG>(a, cs, tile_addr<CONTIG, C, true>(a, launder(tile)));
      }
    }
    __syncthreads();
  }
}

// launch-shape policy per transform length: <= 64 registers per thread,
// >= 32 resident warps per SM where shared memory allows
template <int LOGN>
struct DstShape {
#ifndef FL_NFFT10
#define FL_NFFT10 8
#endif
#ifndef FL_NT10
#define FL_NT10 512
#endif
#ifndef FL_MINB10
#define FL_MINB10 1
#endif
  static constexpr int NFFT =
      LOGN == 10 ? FL_NFFT10 : (LOGN <= 8 ? 16 : (LOGN >= 12 ? 1 : (8 >> (LOGN - 9))));
  static constexpr int NT = LOGN == 10 ? FL_NT10 : (LOGN >= 13 ? 1024 : (LOGN >= 8 ? 512 : (LOGN <= 5 ? 128 : 256)));
  static constexpr int MINB = LOGN == 10 ? FL_MINB10 : (LOGN >= 13 ? 1 : (LOGN >= 8 ? 2 : (LOGN <= 5 ? 8 : 4)));
#ifndef FL_MID_SPLIT
#define FL_MID_SPLIT 0
#endif
#ifndef FL_PLAIN_SPLIT
#define FL_PLAIN_SPLIT 0
#endif
  // optional half-size tiles (NFFT/2 FFTs, NT/2 threads, twice the CTAs):
  // more independent CTAs per SM for the same warp count
  static constexpr bool SPLIT_MID = FL_MID_SPLIT && LOGN >= 8 && LOGN <= 11;
  static constexpr bool SPLIT_PLAIN = FL_PLAIN_SPLIT && LOGN >= 8 && LOGN <= 11;
  static constexpr int NFFT_MID = SPLIT_MID ? NFFT / 2 : NFFT;
  static constexpr int NT_MID = SPLIT_MID ? NT / 2 : NT;
  static constexpr int MINB_MID = SPLIT_MID ? 2 * MINB : MINB;
  static constexpr int NFFT_PLAIN = SPLIT_PLAIN ? NFFT / 2 : NFFT;
  static constexpr int NT_PLAIN = SPLIT_PLAIN ? NT / 2 : NT;
  static constexpr int MINB_PLAIN = SPLIT_PLAIN ? 2 * MINB : MINB;
  static constexpr size_t smem_n(int nt, int nfft) {
    return size_t(16) * (size_t(1) << LOGN) * nfft + size_t(16) * nfft * (nt / 32);
  }
  static constexpr size_t smem(int nt) { return smem_n(nt, NFFT); }
  static constexpr size_t smem_mid(int nt) { return smem_n(nt, NFFT_MID) + GatherTable<LOGN>::bytes(); }
};

}  // namespace fl
