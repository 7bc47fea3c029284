// Warp-per-FFT DST-I pass (same algorithm as dst_fft.cuh, different mapping).
//
// A tile holds C = 2*W lines as W packed complex sequences; warp w owns
// sequence w.  Only the tile-wide phases (coalesced load + pre-processing and
// the coalesced store) need block barriers; the FFT stages and the
// split/scan post-processing touch only the warp's own sequence and run under
// __syncwarp, with the odd-output prefix sum as a warp shuffle scan.
//
// Shared-memory layout: sequence-major cells, cell(p, pos) = p*N + (pos ^ key),
// key = ((pos >> 3) ^ p) & 7: row writes across sequences (load/store), unit
// stride runs and the stride-1 last radix-8 stage are all conflict-free.
#pragma once

#include "dst_fft.cuh"

namespace fl {

template <int LOGN, int W>
struct WCells {
  static constexpr int N = 1 << LOGN;
  double2* D;
  __device__ __forceinline__ static int idx(int p, int pos) {
    if constexpr (LOGN >= 6) return p * N + (pos ^ (((pos >> 3) ^ p) & 7));
    else return p * N + pos;
  }
  __device__ __forceinline__ double& re(int l, int j) const {
    return reinterpret_cast<double*>(D)[2 * idx(l >> 1, j) + (l & 1)];
  }
};

// one DIF (or, with DIT, twiddle-first) stage of sequence p by one warp
template <int LOGN, int W, int LGL, int RL, bool DIT>
__device__ __forceinline__ void wfft_stage(const WCells<LOGN, W>& cs, int p, const double2* __restrict__ tw) {
  using CS = WCells<LOGN, W>;
  constexpr int N = 1 << LOGN;
  constexpr int R = 1 << RL;
  constexpr int LGST = LGL - RL;
  constexpr int ST = 1 << LGST;
  constexpr int NB = N / R;
  constexpr int PER = (NB + 31) / 32;
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int bi = lane + 32 * it;
    if (NB % 32 == 0 || bi < NB) {
      const int j = bi & (ST - 1);
      const int base = ((bi >> LGST) << LGL) + j;
      double2 v[R];
#pragma unroll
      for (int t = 0; t < R; ++t) v[t] = cs.D[CS::idx(p, base + t * ST)];
      if constexpr (DIT && LGST > 0) {
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
      if constexpr (!DIT && LGST > 0) {
#pragma unroll
        for (int q = 1; q < R; ++q) v[q] = cmul(v[q], __ldg(&tw[(j * q) << (LOGN - LGL)]));
      }
#pragma unroll
      for (int q = 0; q < R; ++q) cs.D[CS::idx(p, base + q * ST)] = v[q];
    }
  }
  __syncwarp();
}

template <int LOGN, int W, int S, int LGL>
__device__ __forceinline__ void wfft_rec(const WCells<LOGN, W>& cs, int p, const double2* __restrict__ tw) {
  if constexpr (S < FftPlan<LOGN>::NST) {
    constexpr int RL = FftPlan<LOGN>::rlog(S);
    wfft_stage<LOGN, W, LGL, RL, false>(cs, p, tw);
    wfft_rec<LOGN, W, S + 1, LGL - RL>(cs, p, tw);
  }
}

template <int LOGN, int W, int S>
__device__ __forceinline__ void wdit_rec(const WCells<LOGN, W>& cs, int p, const double2* __restrict__ tw) {
  if constexpr (S >= 0) {
    wfft_stage<LOGN, W, StageLGL<LOGN, S>::value, FftPlan<LOGN>::rlog(S), true>(cs, p, tw);
    wdit_rec<LOGN, W, S - 1>(cs, p, tw);
  }
}

// warp inclusive scan of a double2
__device__ __forceinline__ double2 warp_incl_scan(double2 x) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double yx = __shfl_up_sync(0xffffffffu, x.x, d);
    const double yy = __shfl_up_sync(0xffffffffu, x.y, d);
    if (lane >= d) {
      x.x += yx;
      x.y += yy;
    }
  }
  return x;
}

// post-processing of sequence p by its warp; NAT: spectrum in natural order
template <int LOGN, int W, bool NAT>
__device__ __forceinline__ void wpost(const WCells<LOGN, W>& cs, int p) {
  using CS = WCells<LOGN, W>;
  constexpr int N = 1 << LOGN;
  constexpr int H = N / 2;
  constexpr int G = H < 32 ? H : 32;
  constexpr int K = H / G;
  const int g = threadIdx.x & 31;
  const bool active = g < G;
  const int A = NAT ? g * K : perm_of<LOGN>(g * K);
  const int B = (g == 0) ? 0 : (NAT ? N - g * K : (N - 1 - perm_of<LOGN>(g * K - 1)));
  double2 tot = make_double2(0.0, 0.0);
  if (active) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int ck_pos = NAT ? A + i : (A | perm_c<LOGN>(i));
      const int cm_pos = (i == 0) ? B : (NAT ? N - A - i : (N - 1 - (A | perm_c<LOGN>(i - 1))));
      const int ik = CS::idx(p, ck_pos), im = CS::idx(p, cm_pos);
      const double2 ck = cs.D[ik];
      const double2 cm = cs.D[im];
      const double2 e = make_double2(0.5 * (cm.y - ck.y), 0.5 * (ck.x - cm.x));
      double2 r = make_double2(0.5 * (ck.x + cm.x), 0.5 * (ck.y + cm.y));
      if (i == 0 && g == 0) {
        r.x *= 0.5;
        r.y *= 0.5;
        cs.D[ik] = r;
      } else {
        cs.D[ik] = e;
        cs.D[im] = r;
      }
      tot.x += r.x;
      tot.y += r.y;
    }
  }
  const double2 inc = warp_incl_scan(tot);
  double2 run = make_double2(inc.x - tot.x, inc.y - tot.y);
  if (active) {
#pragma unroll
    for (int i = 0; i < K; ++i) {
      const int cm_pos = (i == 0) ? B : (NAT ? N - A - i : (N - 1 - (A | perm_c<LOGN>(i - 1))));
      const int im = CS::idx(p, cm_pos);
      const double2 r = cs.D[im];
      run.x += r.x;
      run.y += r.y;
      cs.D[im] = run;
    }
  }
  __syncwarp();
}

template <int LOGN, int W, bool NAT>
__device__ __forceinline__ double wpost_val(const WCells<LOGN, W>& cs, int l, int cell) {
  return reinterpret_cast<const double*>(cs.D)[2 * WCells<LOGN, W>::idx(l >> 1, cell) + (l & 1)];
}

// tile-wide load + pre-processing (block mapping of dst_fft.cuh's Split)
template <int LOGN, int W, int NT, bool CONTIG, int LOADER>
__device__ __forceinline__ void wload_pre(const DstArgs& a, const WCells<LOGN, W>& cs, const TileAddr& ta) {
  using SP = Split<LOGN, W, NT, CONTIG>;
  constexpr int N = SP::N, H = SP::H, PER = SP::PER;
  constexpr int B = PER < 8 ? PER : 8;
  static_assert(PER % B == 0, "batch must divide the per-thread item count");
  int k0, l0;
  SP::base(threadIdx.x, k0, l0);
  const double* xp = a.x + ta.base + (int64_t)l0 * ta.LS;
  const double* pa = xp + (int64_t)k0 * ta.JS;
  const double* pb = xp + (int64_t)(N - 2 - k0) * ta.JS;
#pragma unroll
  for (int it0 = 0; it0 < PER; it0 += B) {
    double xa[B], xb[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int it = it0 + u;
      const int l = l0 + SP::LD(it);
      const int k = k0 + SP::MS(it);
      xa[u] = 0.0;
      xb[u] = 0.0;
      if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
        if constexpr (LOADER == LOAD_PLAIN) {
          xa[u] = __ldg(pa + (int64_t)SP::LD(it) * ta.LS + (int64_t)SP::MS(it) * ta.JS);
          if (k + 1 < H) xb[u] = __ldg(pb + (int64_t)SP::LD(it) * ta.LS - (int64_t)SP::MS(it) * ta.JS);
        } else {
          xa[u] = load_elem<LOADER>(a, ta, l, k);
          if (k + 1 < H) xb[u] = load_elem<LOADER>(a, ta, l, N - k - 2);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int it = it0 + u;
      if (SP::ok(threadIdx.x, it)) {
        const int l = l0 + SP::LD(it);
        const int j = k0 + SP::MS(it) + 1;
        if (j == H) {
          cs.re(l, H) = 2.0 * xa[u];
        } else {
          const double s = __ldg(&a.sn[j]);
          const double sum = s * (xa[u] + xb[u]), dif = 0.5 * (xa[u] - xb[u]);
          cs.re(l, j) = sum + dif;
          cs.re(l, N - j) = sum - dif;
        }
      }
    }
  }
  for (int l = threadIdx.x; l < SP::C; l += NT) cs.re(l, 0) = 0.0;
}

// tile-wide store of rows 2k, 2k+1 from cells perm(k), perm(N-k) (or k, N-k)
template <int LOGN, int W, int NT, bool CONTIG, bool NAT>
__device__ __forceinline__ void wstore(const DstArgs& a, const WCells<LOGN, W>& cs, const TileAddr& ta_in) {
  using SP = Split<LOGN, W, NT, CONTIG>;
  const TileAddr ta = ta_in.fresh();
  const double sc = a.scale;
  int k0, l0;
  SP::base(launder((int)threadIdx.x), k0, l0);
  const KCells kc = kcells<LOGN>(k0);
  double* yb = a.y + ta.base + (int64_t)l0 * ta.LS;
#pragma unroll
  for (int it = 0; it < SP::PER; ++it) {
    const int l = l0 + SP::LD(it);
    const int k = k0 + SP::MS(it);
    if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
      double* yl = yb + (int64_t)SP::LD(it) * ta.LS;
      const int ce = NAT ? k : cell_even<LOGN>(kc, SP::MS(it));
      const int co = NAT ? ((SP::N - k) & (SP::N - 1)) : cell_odd<LOGN>(kc, SP::MS(it));
      yl[(int64_t)(2 * k) * ta.JS] = sc * wpost_val<LOGN, W, NAT>(cs, l, co);
      if (k > 0) yl[(int64_t)(2 * k - 1) * ta.JS] = sc * wpost_val<LOGN, W, NAT>(cs, l, ce);
    }
  }
}

// fused pass: in-place core scaling (coalesced store mapping, private cells)
template <int LOGN, int W, int NT, bool CONTIG>
__device__ __forceinline__ void wcore_scale(const DstArgs& a, const WCells<LOGN, W>& cs, const TileAddr& ta_in) {
  using SP = Split<LOGN, W, NT, CONTIG>;
  using CS = WCells<LOGN, W>;
  const TileAddr ta = ta_in.fresh();
  constexpr int PER = SP::PER;
  constexpr int B = PER < 4 ? PER : 4;
  int k0, l0;
  SP::base(threadIdx.x, k0, l0);
  const KCells kc = kcells<LOGN>(k0);
  const double* cb = a.core + ta.base + (int64_t)l0 * ta.LS;
  double* D = reinterpret_cast<double*>(cs.D);
#pragma unroll
  for (int it0 = 0; it0 < PER; it0 += B) {
    double ce_v[B], co_v[B];
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int it = it0 + u;
      const int l = l0 + SP::LD(it);
      const int k = k0 + SP::MS(it);
      ce_v[u] = 0.0;
      co_v[u] = 0.0;
      if (SP::ok(threadIdx.x, it) && l < ta.lmax) {
        const double* cl = cb + (int64_t)SP::LD(it) * ta.LS;
        co_v[u] = __ldg(cl + (int64_t)(2 * k) * ta.JS);
        if (k > 0) ce_v[u] = __ldg(cl + (int64_t)(2 * k - 1) * ta.JS);
      }
    }
#pragma unroll
    for (int u = 0; u < B; ++u) {
      const int it = it0 + u;
      const int l = l0 + SP::LD(it);
      if (SP::ok(threadIdx.x, it)) {
        D[2 * CS::idx(l >> 1, cell_odd<LOGN>(kc, SP::MS(it))) + (l & 1)] *= co_v[u];
        if (k0 + SP::MS(it) > 0) D[2 * CS::idx(l >> 1, cell_even<LOGN>(kc, SP::MS(it))) + (l & 1)] *= ce_v[u];
      }
    }
  }
}

// fused pass: first DIT stage with the DST-I pre-processing gathered from the
// permuted, core-scaled spectrum of the same sequence (warp-private)
template <int LOGN, int W>
__device__ __forceinline__ void wdit_gather(const DstArgs& a, const WCells<LOGN, W>& cs, int p) {
  using CS = WCells<LOGN, W>;
  constexpr int N = 1 << LOGN;
  constexpr int H = N / 2;
  constexpr int RL = FftPlan<LOGN>::rlog(FftPlan<LOGN>::NST - 1);
  constexpr int R = 1 << RL;
  constexpr int NB = N / R;
  constexpr int PER = (NB + 31) / 32;
  const int lane = threadIdx.x & 31;
  double2 v[PER][R];
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int bi = lane + 32 * it;
    if (NB % 32 == 0 || bi < NB) {
      const int base = bi * R;
#pragma unroll
      for (int t = 0; t < R; ++t) {
        const int j = perm_inv<LOGN>(base + t);
        double2 y = make_double2(0.0, 0.0);
        if (j != 0) {
          const double2 xa = cs.D[CS::idx(p, out_pos<LOGN>(j))];
          const double2 xb = (j == H) ? xa : cs.D[CS::idx(p, out_pos<LOGN>(N - j))];
          const double s = __ldg(&a.sn[j < H ? j : N - j]);
          y = make_double2(fma(s, xa.x + xb.x, 0.5 * (xa.x - xb.x)), fma(s, xa.y + xb.y, 0.5 * (xa.y - xb.y)));
        }
        v[it][t] = y;
      }
      dftR<RL>(v[it]);
    }
  }
  __syncwarp();
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int bi = lane + 32 * it;
    if (NB % 32 == 0 || bi < NB) {
#pragma unroll
      for (int q = 0; q < R; ++q) cs.D[CS::idx(p, bi * R + q)] = v[it][q];
    }
  }
  __syncwarp();
}

template <int LOGN, int W, int MINB, bool CONTIG, int LOADER, bool MIDCORE>
__global__ void __launch_bounds__(32 * W, MINB) k_dst_warp(const DstArgs a) {
  using CS = WCells<LOGN, W>;
  constexpr int NT = 32 * W;
  constexpr int C = 2 * W;
  extern __shared__ __align__(16) double smem_dst[];
  const CS cs{reinterpret_cast<double2*>(smem_dst)};
  const int p = threadIdx.x >> 5;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x) {
    wload_pre<LOGN, W, NT, CONTIG, LOADER>(a, cs, tile_addr<CONTIG, C>(a, tile));
    __syncthreads();
    wfft_rec<LOGN, W, 0, LOGN>(cs, p, a.tw);
    wpost<LOGN, W, false>(cs, p);
    if constexpr (MIDCORE) {
      __syncthreads();
      wcore_scale<LOGN, W, NT, CONTIG>(a, cs, tile_addr<CONTIG, C>(a, launder(tile)));
      __syncthreads();
      wdit_gather<LOGN, W>(a, cs, p);
      wdit_rec<LOGN, W, FftPlan<LOGN>::NST - 2>(cs, p, a.tw);
      wpost<LOGN, W, true>(cs, p);
      __syncthreads();
      wstore<LOGN, W, NT, CONTIG, true>(a, cs, tile_addr<CONTIG, C>(a, launder(tile)));
    } else {
      __syncthreads();
      wstore<LOGN, W, NT, CONTIG, false>(a, cs, tile_addr<CONTIG, C>(a, launder(tile)));
    }
    __syncthreads();
  }
}

// warp-per-FFT shape: W warps (= sequences) per CTA, W*N*16 B of smem
template <int LOGN>
struct WarpShape {
  static constexpr bool ENABLED = LOGN >= 6 && LOGN <= 9;
  static constexpr int W = 8;
  static constexpr int MINB = 3;
  static constexpr size_t SMEM = size_t(16) * W * (size_t(1) << LOGN);
};

}  // namespace fl
