// Register-resident DST-I for N = n + 1 = 1024 (n = 1023, configs[3]): the
// N = 512 design of dst_reg.cuh with one packed FFT per warp.
//
//   * 1024 = 32 x 32: lane q (0..31) holds y_{q + 32 m}, m < 32, runs the
//     32-point DFTs in registers, twiddles by W_1024^{q k2}, one warp-private
//     exchange (two rounds of 8 KB) hands lane q column k2 = q for the second
//     32-point DFT; the spectrum staging (two rounds) gives lane q the
//     frequencies k in [16q, 16q + 16) and their partners N - k for the
//     split; the odd outputs are scanned in registers with 5 shuffle levels.
//   * a CTA of 8 warps owns 16 lines (warp w: lines 2w, 2w+1): strided tiles
//     (1024 rows x 128 B) arrive by four TMA boxes and leave by TMA tensor
//     stores in two halves of the rows through the 64 KB of warp scratch;
//     contiguous tiles arrive by one bulk copy per warp (its 2 lines are one
//     aligned blob at pitch 1023 or 1024).  192 KB of shared memory per CTA,
//     one CTA per SM, 255 registers.
// Plain passes only (the fused operator pass at n = 1023 keeps the CTA
// kernel of dst_fft.cuh).
#pragma once

#include "dst_reg.cuh"

namespace fl {
namespace rg10 {

using rg::brev;
using rg::kc;
using rg::ks;
using rg::SIDE_CONTIG;
using rg::SIDE_SCALAR;
using rg::SIDE_VEC;
using rg::Tile;

constexpr int N = 1024, H = 512;
constexpr int NWARP = 8;
constexpr int TILE = 8192;  // double2 (128 KB): 1024 rows x 16 columns
constexpr int SCR = 512;    // double2 per warp scratch (8 KB)

__host__ __device__ constexpr int tidx(int j, int c) { return j * 8 + (c ^ (j & 7)); }

struct Lane {
  int q;
  double sq, cq;             // sin, cos of pi q / 1024
  double2 w1, w8, w16, w24;  // W_1024^{q}, ^{8q}, ^{16q}, ^{24q}
};

__device__ __forceinline__ Lane lane_consts(const DstArgs& a, int lane) {
  Lane c;
  c.q = lane;
  c.sq = rg::ld_opaque(a.sn + c.q);
  c.cq = rg::ld_opaque(a.sn + H - c.q);
  c.w1 = rg::ld_opaque2(a.tw + c.q);
  c.w8 = rg::ld_opaque2(a.tw + 8 * c.q);
  c.w16 = rg::ld_opaque2(a.tw + 16 * c.q);
  c.w24 = rg::ld_opaque2(a.tw + 24 * c.q);
  return c;
}

// sc * y_j, j = q + 32 m (sin(pi j / 1024) = sin(pi q / 1024 + pi m / 32))
__device__ __forceinline__ double2 pre_y(const Lane& c, int m, double2 xa, double2 xb, double sc, double hsc) {
  const double s = fma(c.sq, kc(m), c.cq * ks(m));
  const double sp = fma(s, sc, hsc), sm = fma(s, sc, -hsc);
  double2 y = make_double2(fma(sp, xa.x, sm * xb.x), fma(sp, xa.y, sm * xb.y));
  if (m == 0 && c.q == 0) y = make_double2(0.0, 0.0);
  if (m == 16 && c.q == 0) y = make_double2((sc + sc) * xa.x, (sc + sc) * xa.y);
  return y;
}

template <bool CONTIG>
__device__ __forceinline__ void pre_read(const double2* tile, int w, const Lane& c_in, double2 (&v)[32], double sc,
                                         int sha, int shb, int sp) {
  Lane c = c_in;
  const int q = c.q, q7 = q & 7;
  const double hsc = 0.5 * sc;
  auto batch = [&](int m) {
    if (m % 8 == 0) {
      rg::sched_fence();
      c.sq = rg::launder_d(c.sq);
      c.cq = rg::launder_d(c.cq);
    }
  };
  if constexpr (CONTIG) {
    const double* d = reinterpret_cast<const double*>(tile) + w * 2048;  // lines 2w (real), 2w + 1 (imag)
    const double* ra = d + sha - 1;
    const double* rb = d + sp + shb - 1;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      batch(m);
      const int j = (m == 0) ? (q == 0 ? 1 : q) : q + 32 * m;
      const int jp = N - q - 32 * m;
      const int jb = (m == 0 && q == 0) ? 1 : jp;
      v[m] = pre_y(c, m, make_double2(ra[j], rb[j]), make_double2(ra[jb], rb[jb]), sc, hsc);
    }
  } else {
    const int ch = w;
    const int la = tidx(q, ch);                                              // + 256 m
    const int lb = q == 0 ? 256 + ch : (32 - q) * 8 + (ch ^ ((8 - q7) & 7));  // + 256 (31 - m)
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      batch(m);
      const int ia = la + 256 * m;
      const int ib = (m == 0 && q == 0) ? la : lb + 256 * (31 - m);
      v[m] = pre_y(c, m, tile[ia], tile[ib], sc, hsc);
    }
  }
}

#ifndef FL_R10_XTILE
#define FL_R10_XTILE 1
#endif

// First half of lane q's FFT: 32-point DFTs, twiddles, the transpose and the
// second 32-point DFTs; w[i] = X[q + 32 brev(i)].  XTILE: the transpose runs
// in one round through a 16 KB buffer xb (the warp's slice of the consumed
// input tile), so a lane never holds more than its 32 values; otherwise two
// rounds through the 8 KB scratch sf (readers then hold 16 unwritten values
// plus 32 received, which spills).
template <bool XTILE>
__device__ __forceinline__ void fft_a(double2* xb, double2* sf, const Lane& c, double2 (&v)[32],
                                      double2 (&w)[32]) {
  const int q = c.q;
  rg::dif<32>(v);
  if constexpr (XTILE) {
    // entry (k2, q') at k2 * 32 + (q' ^ (k2 & 7))
#pragma unroll
    for (int h = 0; h < 4; ++h) {
      double2 t = h == 1 ? c.w8 : h == 2 ? c.w16 : c.w24;
#pragma unroll
      for (int l = 0; l < 8; ++l) {
        const int k2 = 8 * h + l;
        double2 val = v[brev(k2, 5)];
        if (h == 0 && l == 1) t = c.w1;
        if ((h == 0 && l >= 2) || (h > 0 && l >= 1)) t = cmul(t, c.w1);
        if (k2) val = cmul(val, t);
        xb[k2 * 32 + (q ^ (k2 & 7))] = val;
      }
    }
    __syncwarp();
#pragma unroll
    for (int qq = 0; qq < 32; ++qq) w[qq] = xb[q * 32 + (qq ^ (q & 7))];
  } else {
    // two rounds of k2: entry (kk, q') at kk * 32 + (q' ^ (kk & 7))
#pragma unroll
    for (int rd = 0; rd < 2; ++rd) {
#pragma unroll
      for (int hh = 0; hh < 2; ++hh) {
        const int h = 2 * rd + hh;
        double2 t = h == 1 ? c.w8 : h == 2 ? c.w16 : c.w24;
#pragma unroll
        for (int l = 0; l < 8; ++l) {
          const int k2 = 8 * h + l;
          double2 val = v[brev(k2, 5)];
          if (h == 0 && l == 1) t = c.w1;
          if ((h == 0 && l >= 2) || (h > 0 && l >= 1)) t = cmul(t, c.w1);
          if (k2) val = cmul(val, t);
          const int kk = k2 & 15;
          sf[kk * 32 + (q ^ (kk & 7))] = val;
        }
      }
      __syncwarp();
      if ((q >> 4) == rd) {
        const int kk = q & 15;
#pragma unroll
        for (int qq = 0; qq < 32; ++qq) w[qq] = sf[kk * 32 + (qq ^ (kk & 7))];
      }
      __syncwarp();
    }
  }
  rg::dif<32>(w);  // w[i] = X[q + 32 brev(i)]
}

// Second half: spectrum staging, split and scan; ev[i] = S'_{2k},
// od[i] = S'_{2k+1}, k = 16q + i (scaled: the pass's scale rode on the
// pre-processing)
__device__ __forceinline__ void fft_b(double2* sf, const Lane& c, double2 (&w)[32], double2 (&ev)[16],
                                      double2 (&od)[16]) {
  const int q = c.q, q7 = q & 7;
  // spectrum staging in two rounds (k < 512, k >= 512): kk = k mod 512 at
  // kk ^ ((kk >> 4) & 7)
  double2 ck[16], cm[16];
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
#pragma unroll
    for (int i = 0; i < 32; ++i) {
      const int k1 = brev(i, 5);
      if ((k1 >> 4) != rd) continue;
      const int kk = q + 32 * (k1 & 15);
      sf[kk ^ ((kk >> 4) & 7)] = w[i];
    }
    __syncwarp();
    if (rd == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) ck[i] = sf[16 * q + (i ^ q7)];
    } else {
      // partner N - k of k = 16q + i: kk = 16 (31 - q) + (16 - i) for i >= 1,
      // 16 (32 - q) for i = 0 (q >= 1); k = 0 pairs with itself
#pragma unroll
      for (int i = 1; i < 16; ++i) cm[i] = sf[16 * (31 - q) + ((16 - i) ^ ((7 - q7) & 7))];
      cm[0] = q == 0 ? ck[0] : sf[16 * (32 - q) + ((32 - q) & 7)];
    }
    __syncwarp();
  }
  double2 run = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double2 r = make_double2(ck[i].x + cm[i].x, ck[i].y + cm[i].y);
    ev[i] = make_double2(cm[i].y - ck[i].y, ck[i].x - cm[i].x);
    if (i == 0 && q == 0) r = ck[0];
    run.x += r.x;
    run.y += r.y;
    od[i] = run;
  }
  double2 inc = run;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const double ux = __shfl_up_sync(0xffffffffu, inc.x, d);
    const double uy = __shfl_up_sync(0xffffffffu, inc.y, d);
    if (q >= d) {
      inc.x += ux;
      inc.y += uy;
    }
  }
  const double2 off = make_double2(inc.x - run.x, inc.y - run.y);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    od[i].x += off.x;
    od[i].y += off.y;
  }
}

// ---- loads ------------------------------------------------------------------
__device__ __forceinline__ void tma_issue(const DstArgs& a, const CUtensorMap* map, uint32_t t, double2* tile,
                                          uint64_t* bar) {
  const uint32_t o = a.div_blk.div(t);
  const uint32_t r = t - o * a.div_blk.d;
  const uint32_t g = a.div_chunk.div(r);
  const int c0 = (int)(r - g * a.div_chunk.d) * 16;
  mbar_expect_tx(bar, (uint32_t)(TILE * sizeof(double2)));
#pragma unroll
  for (int b = 0; b < 4; ++b) tma_load_4d(tile + b * (TILE / 4), map, c0, 256 * b - 1, (int)g, (int)o, bar);
}

__device__ __forceinline__ bool contig_bulk10(const DstArgs& a, const Tile& tl, int w) {
  return (tl.LS == 1023 || tl.LS == 1024) && 2 * w + 1 < tl.lmax && ((reinterpret_cast<uintptr_t>(a.x) & 15) == 0);
}

// warp w's 2 lines: one bulk copy, or cp.async with per-line shift / zero fill
// (wl: the warp's smem slot, wg: its line pair 2 wg, 2 wg + 1 in the 16-line tile)
__device__ __forceinline__ void issue_contig(const DstArgs& a, uint32_t t, double2* tile, uint32_t stile, int wl,
                                             int wg, int lane, uint64_t* wbar) {
  const Tile tl = rg::tile_of<SIDE_CONTIG, false>(a, t);
  if ((FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) return;
  if (contig_bulk10(a, tl, wg)) {
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)(2 * tl.LS * sizeof(double));
      mbar_expect_tx(wbar, bytes);
      rg::bulk_load(tile + 1024 * wl, a.x + tl.base + (int64_t)(2 * wg) * tl.LS, bytes, wbar);
    }
    return;
  }
  const uint32_t d = stile + 8u * (uint32_t)(wl * 2048) + 16u * (uint32_t)lane;
  rg::static_for<0, 2>([&](auto L) {
    constexpr int l = decltype(L)::value;
    const bool ok = 2 * wg + l < tl.lmax;
    const int sh = ok ? rg::line_shift(tl, 2 * wg + l) : 0;
    const double* src = ok ? a.x + tl.base + (int64_t)(2 * wg + l) * tl.LS - sh + 2 * lane : a.x;
    const int sz = ok ? 16 : 0;
    const int szl = ok ? (sh ? 16 : (lane == 31 ? 8 : 16)) : 0;
    rg::static_for<0, 16>([&](auto I) {
      constexpr int i = decltype(I)::value;
      rg::cp16<8 * (l * 1024 + 64 * i)>(d, ok ? src + 64 * i : a.x, i == 15 ? szl : sz);
    });
  });
}

// ---- stores -----------------------------------------------------------------
// TMA tensor stores: g = r - 1 = 32 qq + ii, staging [ii][qq][16 columns];
// half 0 = qq 0..15 (box {16, 16, 32}), half 1 = qq 16..30 ({16, 15, 32})
// and qq 31 with 31 rows ({16, 1, 31})
__device__ __forceinline__ int stg_idx(int hh, int qq, int ii, int ch) {
  if (hh == 0) {
    const int R = ii * 16 + qq;
    return R * 8 + (ch ^ (R & 7));
  }
  if (qq < 31) {
    const int R = ii * 15 + (qq - 16);
    return R * 8 + (ch ^ (R & 7));
  }
  return 3840 + ii * 8 + (ch ^ (ii & 7));
}

__device__ __forceinline__ void store_strided_tma(const DstArgs& a, const rg::OutMaps* maps, uint32_t t, double2* stg,
                                                  int w, int q, const double2 (&ev)[16], const double2 (&od)[16]) {
  const int ch = w;
  const uint32_t o = a.div_blk.div(t);
  const uint32_t rr = t - o * a.div_blk.d;
  const uint32_t g = a.div_chunk.div(rr);
  const int c0 = (int)(rr - g * a.div_chunk.d) * 16;
  __syncthreads();  // the staging spans every warp's scratch
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    if ((q >> 4) == hh) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i > 0) stg[stg_idx(hh, q, 2 * i - 1, ch)] = ev[i];
        stg[stg_idx(hh, q, 2 * i, ch)] = od[i];
      }
    }
    if (q >= 1 && ((q - 1) >> 4) == hh) stg[stg_idx(hh, q - 1, 31, ch)] = ev[0];
    rg::proxy_fence_async();
    __syncthreads();
    if (threadIdx.x == 0 && !(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 3)) {
      if (hh == 0) {
        rg::tma_store_5d(&maps->a, stg, c0, 0, 0, (int)g, (int)o);
      } else {
        rg::tma_store_5d(&maps->b, stg, c0, 16, 0, (int)g, (int)o);
        rg::tma_store_5d(&maps->c, stg + 3840, c0, 31, 0, (int)g, (int)o);
      }
      rg::bulk_commit();
      if (hh == 0) rg::bulk_wait_read();
    }
    // half 1's staging is reread by the TMA engine while the next tile is
    // pre-read; the kernel waits for it before the next exchange
    if (hh == 0) __syncthreads();
  }
}

// contiguous output of warp w (lines 2w, 2w + 1) through its 8 KB scratch in
// two halves of positions p = r - 1: [0, 512), [512, 1024) (1023 is padding)
__device__ __forceinline__ int cstg(int p) { return (((p >> 1) ^ ((p >> 5) & 7)) << 1) | (p & 1); }

__device__ __forceinline__ void store_contig(const DstArgs& a, uint32_t t, double2* scr, int w, int lane,
                                             const double2 (&ev)[16], const double2 (&od)[16]) {
  const int q = lane;
  const Tile tl = rg::tile_of<SIDE_CONTIG, true>(a, t);
  double* sd = reinterpret_cast<double*>(scr);
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    if ((q >> 4) == hh) {
      const int base = 32 * (q - 16 * hh);
#pragma unroll
      for (int i = 0; i < 15; ++i) {
        const int ph = cstg(base + 2 * i);
        *reinterpret_cast<double2*>(sd + ph) = make_double2(od[i].x, ev[i + 1].x);
        *reinterpret_cast<double2*>(sd + 512 + ph) = make_double2(od[i].y, ev[i + 1].y);
      }
      sd[cstg(base + 30)] = od[15].x;
      sd[512 + cstg(base + 30)] = od[15].y;
    }
    if (q >= 1 && ((q - 1) >> 4) == hh) {
      const int pl = 32 * q - 1 - 512 * hh;
      sd[cstg(pl)] = ev[0].x;
      sd[512 + cstg(pl)] = ev[0].y;
    }
    __syncwarp();
#pragma unroll
    for (int l = 0; l < 2; ++l) {
      if (2 * w + l < tl.lmax && (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 3) || a.scale == 12345.0)) {
        const int64_t off = tl.base + (int64_t)(2 * w + l) * tl.LS + 512 * hh;
        const bool al = ((off & 1) == 0) && ((reinterpret_cast<uintptr_t>(a.y) & 15) == 0);
        double* y = a.y + off;
#pragma unroll
        for (int s = 0; s < 8; ++s) {
          const int c = lane + 32 * s;
          const double2 val = *reinterpret_cast<const double2*>(sd + l * 512 + 2 * (c ^ ((c >> 4) & 7)));
          const bool last = (hh == 1 && c == 255);
          if (al && (!last || a.pad_zero)) {
            *reinterpret_cast<double2*>(y + 2 * c) = last ? make_double2(val.x, 0.0) : val;
          } else {
            y[2 * c] = val.x;
            if (!last) y[2 * c + 1] = val.y;
            else if (a.pad_zero) y[2 * c + 1] = 0.0;
          }
        }
      }
    }
    __syncwarp();
  }
}

// Persistent CTAs of NW warps.  Strided: NW = 8, one 16-line tile at a time,
// one CTA per SM.  Contiguous: NW = 8 or 4; with 4, a CTA takes one half
// (8 lines) of a 16-line tile at a time and two CTAs share an SM, so one's
// stores overlap the other's FFTs.
template <int SIDE_IN, int NW>
__global__ void __launch_bounds__(32 * NW, 8 / NW) k_dst_reg10(const DstArgs a, const __grid_constant__ CUtensorMap map,
                                                               const __grid_constant__ rg::OutMaps omaps) {
  static_assert(NW == 8 || (NW == 4 && SIDE_IN == SIDE_CONTIG), "strided tiles need 8 warps");
  constexpr uint32_t PIECES = 8 / NW;  // CTA pieces per 16-line tile
  extern __shared__ __align__(1024) double2 smem10[];
  double2* const tile = smem10;
  double2* const scr_all = smem10 + NW * 1024;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(scr_all + NW * SCR);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint64_t* const wbar = bar + 1 + w;
  double2* const scr = scr_all + SCR * w;
  const uint32_t stile = smem_u32(tile);
  const uint32_t ntiles = (uint32_t)a.ntiles * PIECES;
  constexpr bool STRIDED = SIDE_IN != SIDE_CONTIG;
  if (STRIDED && (stile & 1023u) != 0) __trap();
  if (threadIdx.x == 0) mbar_init(bar, 1);
  if (lane == 0) mbar_init(wbar, 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  uint32_t phase = 0, wphase = 0;
  uint32_t t = blockIdx.x;
  auto issue_next = [&](uint32_t tt) {
    if constexpr (STRIDED) {
      if (threadIdx.x == 0 && !(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) tma_issue(a, &map, tt, tile, bar);
    } else {
      issue_contig(a, tt / PIECES, tile, stile, w, w + NW * (int)(tt % PIECES), lane, wbar);
    }
  };
  if (t < ntiles) issue_next(t);
  rg::cp_commit();
  for (; t < ntiles; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
    int sha = 0, shb = 0, sp = 1024;
    const uint32_t tt = t / PIECES;                 // 16-line tile
    const int wg = w + NW * (int)(t % PIECES);      // line pair in it
    if constexpr (STRIDED) {
      if (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) mbar_wait(bar, phase);
      phase ^= 1;
    } else {
      const Tile tin = rg::tile_of<SIDE_CONTIG, false>(a, tt);
      if (contig_bulk10(a, tin, wg)) {
        if (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) mbar_wait(wbar, wphase);
        wphase ^= 1;
        sp = (int)tin.LS;
      } else {
        sha = rg::line_shift(tin, 2 * wg);
        shb = rg::line_shift(tin, 2 * wg + 1);
      }
    }
    rg::cp_wait<0>();
    // strided tiles arrive by TMA and every thread waited on the mbarrier
    if constexpr (!STRIDED) __syncwarp();
    double2 v[32], wv[32], ev[16], od[16];
    const Lane c = lane_consts(a, lane);
    pre_read<!STRIDED>(tile, w, c, v, 0.5 * a.scale, sha, shb, sp);
    if constexpr (FL_R10_XTILE) {
      // the tile is consumed: warp w's 16 KB slice of it carries the
      // transpose, then the next tile is issued into it
      if (STRIDED) __syncthreads(); else __syncwarp();
      fft_a<true>(tile + 1024 * w, scr, c, v, wv);
      rg::proxy_fence_async();
      if (STRIDED && threadIdx.x == 0) rg::bulk_wait_read();  // previous tile's half-1 store
      if (STRIDED) __syncthreads(); else __syncwarp();
      if (tn < ntiles) issue_next(tn);
      rg::cp_commit();
    } else {
      rg::proxy_fence_async();
      if (STRIDED && threadIdx.x == 0) rg::bulk_wait_read();  // previous tile's half-1 store
      if (STRIDED) __syncthreads(); else __syncwarp();
      if (tn < ntiles) issue_next(tn);
      rg::cp_commit();
      fft_a<false>(nullptr, scr, c, v, wv);
    }
    fft_b(scr, c, wv, ev, od);
    if constexpr (STRIDED) {
      store_strided_tma(a, &omaps, t, scr_all, w, lane, ev, od);
    } else {
      store_contig(a, tt, scr, wg, lane, ev, od);
    }
  }
  rg::cp_wait<0>();
  if (STRIDED && threadIdx.x == 0) rg::bulk_wait_all();
}

template <int NW>
constexpr size_t smem_bytes() { return (size_t)(NW * 1024 + NW * SCR + 8) * sizeof(double2); }

#ifndef FL_R10_CNW
#define FL_R10_CNW 4
#endif
constexpr int CONTIG_NW = FL_R10_CNW;

}  // namespace rg10
}  // namespace fl
