// Register-resident DST-I for N = n + 1 = 512 (the configs[2] grid, n = 511).
//
// Same algorithm as dst_fft.cuh (pre-processing y_j = s_j (x_j + x_{N-j}) +
// (x_j - x_{N-j})/2, two lines per complex FFT, split + segmented scan), but
// the transform itself lives in registers:
//   * a warp owns 4 lines (2 packed complex FFTs, 16 lanes each); lane q
//     holds y_{q + 16 m}, m < 32, and runs the 32-point DFTs in registers;
//     after the W_512^{q k2} twiddles one warp-private shared-memory exchange
//     hands lane q the columns k2 = q and q + 16 for the 16-point DFTs
//     (N = 512 = 32 x 16); a second warp-private staging puts the spectrum in
//     natural order so that lane q splits k in [16q, 16q + 16) against N - k
//     and scans its 16 Re Y values in registers (cross-lane offsets by 4
//     shuffles).  No CTA barrier inside the FFT.
//   * global traffic is organised per CTA of 4 warps = 16 lines: on strided
//     layouts every access covers whole 128-byte row segments (a warp's own
//     4 columns are only 32 bytes of a row; 32-byte accesses cost 1.8-2.5x
//     the DRAM bytes and stall the LSU).  Strided tiles (64 KB, rows of 16
//     columns, 16-byte chunks XOR-swizzled by row = the TMA 128-byte
//     pattern) arrive by two TMA boxes on an mbarrier (cp.async where the
//     side is not 16-byte aligned); the next tile is requested as soon as
//     the current one has been read into registers, so it lands during the
//     FFTs.  Strided outputs leave by TMA tensor stores from a staging in
//     the warps' scratch (a 5-D box that makes the staging conflict-free,
//     see store_strided_tma); contiguous lines by warp-local cp.async loads
//     and 16-byte staged stores.
//   * the fused pass (forward, core, inverse) brings the unit's lane-ordered
//     core slice into the warp's quarter of the consumed tile during the
//     forward FFT and runs the inverse from z written over it.
//   * 96 KB of shared memory per CTA, 2 CTAs per SM, up to 255 registers.
// Every shared-memory and global access is a per-lane base plus a
// compile-time offset; sines and twiddles come from per-lane constants, the
// pass's output scale rides on the pre-processing coefficients.
// Compute-only (no global traffic) the plain pass runs in 0.32 ms at n = 511
// (the CTA kernel of dst_fft.cuh: 0.47 ms); with traffic 0.40 ms strided,
// 0.44 ms contiguous, 0.82 ms fused.
#pragma once

#include <type_traits>

#include "dst_fft.cuh"
#include "tma_util.cuh"

namespace fl {
namespace rg {

constexpr int N = 512, H = 256;
#ifndef FL_REG_PRE_BATCH
#define FL_REG_PRE_BATCH 8
#endif
constexpr int PRE_BATCH = FL_REG_PRE_BATCH;

// unit sides: 16-byte line pairs on a strided layout, single lines on a
// strided layout, contiguous lines with an even pitch
enum { SIDE_VEC = 0, SIDE_SCALAR = 1, SIDE_CONTIG = 2 };
// shared-memory tile layouts read by the pre-processing
enum { RAW_STRIDED = 0, RAW_Z = 1, RAW_CONTIG = 2 };

__host__ __device__ constexpr int brev(int v, int bits) {
  int r = 0;
  for (int b = 0; b < bits; ++b) r |= ((v >> b) & 1) << (bits - 1 - b);
  return r;
}

// cos(pi m / 32), m in [0, 64), from correctly rounded first-quadrant values
__host__ __device__ constexpr double c64(int m) {
  constexpr double t[17] = {1.0,
                            0.9951847266721969,
                            0.9807852804032304,
                            0.9569403357322088,
                            0.9238795325112867,
                            0.881921264348355,
                            0.8314696123025452,
                            0.773010453362737,
                            0.7071067811865476,
                            0.6343932841636455,
                            0.5555702330196022,
                            0.47139673682599764,
                            0.3826834323650898,
                            0.2902846772544624,
                            0.19509032201612828,
                            0.0980171403295606,
                            0.0};
  m &= 63;
  return m <= 16 ? t[m] : m <= 32 ? -t[32 - m] : m <= 48 ? -t[m - 32] : t[64 - m];
}
// sin(pi m / 32)
__host__ __device__ constexpr double s64(int m) { return c64(16 - m); }

// The same values in constant memory: with a compile-time index they are
// constant-bank operands of DFMA/DMUL, whereas FP64 literals are materialised
// in registers and hoisted out of the unit loop (which spills).
#define FL_C64_4(b) c64(b), c64(b + 1), c64(b + 2), c64(b + 3)
#define FL_C64_16(b) FL_C64_4(b), FL_C64_4(b + 4), FL_C64_4(b + 8), FL_C64_4(b + 12)
__constant__ double kcos64[64] = {FL_C64_16(0), FL_C64_16(16), FL_C64_16(32), FL_C64_16(48)};
#undef FL_C64_16
#undef FL_C64_4
__device__ __forceinline__ double kc(int m) { return kcos64[m & 63]; }
__device__ __forceinline__ double ks(int m) { return kcos64[(16 - m) & 63]; }

// x * W_32^e, W_32 = exp(-2 pi i / 32); e is a compile-time constant after
// unrolling, so every branch but one folds away
__device__ __forceinline__ double2 mulw(double2 x, int e) {
  constexpr double r = 0.70710678118654752440084436210485;
  e &= 31;
  if (e == 0) return x;
  if (e == 8) return make_double2(x.y, -x.x);
  if (e == 16) return make_double2(-x.x, -x.y);
  if (e == 24) return make_double2(-x.y, x.x);
  if (e == 4) return make_double2((x.x + x.y) * r, (x.y - x.x) * r);
  if (e == 12) return make_double2((x.y - x.x) * r, -(x.x + x.y) * r);
  if (e == 20) return make_double2(-(x.x + x.y) * r, (x.x - x.y) * r);
  if (e == 28) return make_double2((x.x - x.y) * r, (x.x + x.y) * r);
  const double c = kc(2 * e), s = ks(2 * e);
  return make_double2(fma(x.x, c, x.y * s), fma(x.y, c, -x.x * s));
}

// in-register radix-2 DIF FFT, LEN <= 32: v[i] ends up holding X[brev(i)]
template <int LEN>
__device__ __forceinline__ void dif(double2 (&v)[LEN]) {
#pragma unroll
  for (int half = LEN / 2; half >= 1; half >>= 1) {
#pragma unroll
    for (int b = 0; b < LEN; b += 2 * half) {
#pragma unroll
      for (int j = 0; j < half; ++j) {
        const double2 p = v[b + j], c = v[b + j + half];
        v[b + j] = cadd(p, c);
        v[b + j + half] = mulw(csub(p, c), j * (32 / (2 * half)));
      }
    }
  }
}

// ---- shared-memory layouts ------------------------------------------------
// CTA tile, strided passes: row j (1..511) of the 16 tile columns as 8
// double2 chunks (columns 2c, 2c+1), chunk c stored at c ^ (j & 7)
// (the TMA 128-byte swizzle pattern): 8 consecutive rows of one chunk hit 8
// bank groups.  CTA tile, contiguous passes: [line][512] doubles, row j at j-1.
constexpr int TILE = 4096;   // double2 (64 KB)
constexpr int SCR = 512;     // double2 per warp scratch (8 KB)
constexpr int NWARP = 4;

__host__ __device__ constexpr int tidx(int j, int c) { return j * 8 + (c ^ (j & 7)); }
// z layout of the fused pass (a warp's 16 KB of the tile): double2 (lines
// 2f, 2f+1) of row j at 2j + (f ^ bit 2 of j), low three bits XOR bits 5..7 of
// j: rows q + 16 m (read) and rows 32 apart (written together) are both
// conflict-free
__host__ __device__ constexpr int zidx(int j, int f) { return (2 * j + (f ^ ((j >> 2) & 1))) ^ ((j >> 5) & 7); }
// output staging of strided passes (a warp's scratch, rows r' in [0, 256)):
// zidx pattern, XOR 2w so that the 8 chunks of one row, read across the 4
// warps' scratch, land in 8 bank groups
__host__ __device__ constexpr int sidx(int r, int f, int w) { return zidx(r, f) ^ (2 * w); }

struct Tile {
  int64_t base;   // element offset of (row 1, column / line 0)
  int64_t JS, LS;
  int lmax;       // valid columns / lines of the tile (<= 16)
};

template <int SIDE, bool OUT>
__device__ __forceinline__ Tile tile_of(const DstArgs& a, uint32_t t) {
  Tile r;
  if (SIDE == SIDE_CONTIG) {
    const int64_t L0 = (int64_t)t * 16;
    const int64_t lp = OUT ? a.out_lp : a.in_lp;
    r.base = L0 * lp;
    r.JS = 1;
    r.LS = lp;
    const int64_t rem = a.outer - L0;
    r.lmax = (int)(rem < 16 ? rem : 16);
  } else {
    const uint32_t o = a.div_blk.div(t);
    const uint32_t rr = t - o * a.div_blk.d;
    const uint32_t g = a.div_chunk.div(rr);
    const int64_t c0 = (int64_t)(rr - g * a.div_chunk.d) * 16;
    r.base = (int64_t)o * (OUT ? a.out_os : a.in_os) + (int64_t)g * (OUT ? a.out_gp : a.in_gp) + c0;
    r.JS = OUT ? a.out_js : a.in_js;
    r.LS = 1;
    const int64_t rem = a.wv - c0;
    r.lmax = (int)(rem < 16 ? rem : 16);
  }
  return r;
}


// cp.async with a compile-time shared-memory offset; sz = 0 zero-fills
template <int OFF>
__device__ __forceinline__ void cp16(uint32_t dst, const void* src, int sz) {
  asm volatile("cp.async.cg.shared.global [%0+%3], [%1], 16, %2;\n" ::"r"(dst), "l"(src), "r"(sz), "n"(OFF) : "memory");
}
template <int OFF>
__device__ __forceinline__ void cp8(uint32_t dst, const void* src, int sz) {
  asm volatile("cp.async.ca.shared.global [%0+%3], [%1], 8, %2;\n" ::"r"(dst), "l"(src), "r"(sz), "n"(OFF) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int K>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(K) : "memory");
}

// generic <-> async proxy fence for this CTA's shared memory
__device__ __forceinline__ void proxy_fence_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// compiler-only fence: keeps the scheduler from hoisting a whole phase's
// loads (64 x 16 B in flight would need every register)
__device__ __forceinline__ void sched_fence() { asm volatile("" ::: "memory"); }

template <int I, int END, class F>
__device__ __forceinline__ void static_for(F&& f) {
  if constexpr (I < END) {
    f(std::integral_constant<int, I>{});
    static_for<I + 1, END>(f);
  }
}

#ifndef FL_REG_NOMEM
#define FL_REG_NOMEM 0
#endif

// cp.async loads of strided tile t into the CTA tile (all 4 warps; every
// instruction covers 4 (16-byte side) or 2 (8-byte side) whole row segments)
template <int SIDE>
__device__ __forceinline__ void issue_strided(const DstArgs& a, uint32_t t, uint32_t stile, int w, int lane) {
  if (FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2) return;
  const Tile tl = tile_of<SIDE, false>(a, t);
  if constexpr (SIDE == SIDE_VEC) {
    const int rho = lane >> 3, c = lane & 7;
    const int j0 = 1 + rho + 4 * w;  // rows j0 + 16 s
    const uint32_t d = stile + 16u * (uint32_t)tidx(j0, c);
    const int sz = 2 * c < tl.lmax ? 16 : 0;
    // zero-filled chunks read nothing; their source stays at a.x
    const double* src = sz ? a.x + tl.base + (int64_t)(j0 - 1) * tl.JS + 2 * c : a.x;
    const int64_t step = sz ? 16 * tl.JS : 0;
    static_for<0, 32>([&](auto I) {
      constexpr int s = decltype(I)::value;
      if (s < 31 || j0 < 16) cp16<16 * 128 * s>(d, src, sz);
      src += step;
    });
  } else {
    const int rho = lane >> 4, cc = lane & 15;
    const int j0 = 1 + rho + 2 * w;  // rows j0 + 8 s
    const uint32_t d = stile + 8u * (uint32_t)(2 * tidx(j0, cc >> 1) + (cc & 1));
    const int sz = cc < tl.lmax ? 8 : 0;
    const double* src = sz ? a.x + tl.base + (int64_t)(j0 - 1) * tl.JS + cc : a.x;
    const int64_t step = sz ? 8 * tl.JS : 0;
    static_for<0, 64>([&](auto I) {
      constexpr int s = decltype(I)::value;
      if (s < 63 || j0 < 8) cp8<8 * 128 * s>(d, src, sz);
      src += step;
    });
  }
}

// cp.async loads of warp w's 4 lines of contiguous tile t ([line][512]).
// A line whose start is not 16-byte aligned (odd pitch, e.g. the dense
// 511-pitch tensor) is copied from one element earlier: row j sits at
// position j - 1 + shift, shift = parity of the line's element offset.  The
// last chunk of an aligned line reads only its first element (the second
// would be past the line, possibly past the tensor).
__device__ __forceinline__ int line_shift(const Tile& tl, int l) { return (int)((tl.base + l * tl.LS) & 1); }

__device__ __forceinline__ void issue_contig_tile(const double* x, const Tile& tl, uint32_t stile, int w, int lane) {
  if (FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2) return;
  const uint32_t d = stile + 8u * (uint32_t)(4 * w * 512) + 16u * (uint32_t)lane;
  static_for<0, 4>([&](auto L) {
    constexpr int l = decltype(L)::value;
    const bool ok = 4 * w + l < tl.lmax;
    const int sh = line_shift(tl, 4 * w + l);
    const double* src = ok ? x + tl.base + (int64_t)(4 * w + l) * tl.LS - sh + 2 * lane : x;
    const int sz = ok ? 16 : 0;
    const int szl = ok ? (sh ? 16 : (lane == 31 ? 8 : 16)) : 0;
    static_for<0, 8>([&](auto I) {
      constexpr int i = decltype(I)::value;
      cp16<8 * (l * 512 + 64 * i)>(d, ok ? src + 64 * i : x, i == 7 ? szl : sz);
    });
  });
}

__device__ __forceinline__ void issue_contig(const DstArgs& a, uint32_t t, uint32_t stile, int w, int lane) {
  issue_contig_tile(a.x, tile_of<SIDE_CONTIG, false>(a, t), stile, w, lane);
}

// A warp's 4 lines as one bulk copy when they are one contiguous,
// 16-byte aligned blob: pitch 512 (padded, 16 KB) or the dense pitch 511
// (16352 B; the blob starts at line 16t + 4w, an even line, so at a 16-byte
// aligned offset).  The ragged last tile keeps cp.async (zero fill).
__device__ __forceinline__ bool contig_bulk_p(const double* x, const Tile& tl, int w) {
  return (tl.LS == 511 || tl.LS == 512) && 4 * w + 3 < tl.lmax && ((reinterpret_cast<uintptr_t>(x) & 15) == 0) &&
         ((tl.base + (int64_t)(4 * w) * tl.LS) & 1) == 0;
}
__device__ __forceinline__ bool contig_bulk(const DstArgs& a, const Tile& tl, int w) { return contig_bulk_p(a.x, tl, w); }

__device__ __forceinline__ void bulk_load(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

// contiguous tile issue: bulk copy (lane 0, completes on wbar) or cp.async
__device__ __forceinline__ void issue_contig_any_tile(const double* x, const Tile& tl, double2* tile, uint32_t stile,
                                                      int w, int lane, uint64_t* wbar) {
  if (contig_bulk_p(x, tl, w)) {
    if (lane == 0 && !(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) {
      const uint32_t bytes = (uint32_t)(4 * tl.LS * sizeof(double));
      mbar_expect_tx(wbar, bytes);
      bulk_load(tile + 1024 * w, x + tl.base + (int64_t)(4 * w) * tl.LS, bytes, wbar);
    }
  } else {
    issue_contig_tile(x, tl, stile, w, lane);
  }
}
__device__ __forceinline__ void issue_contig_any(const DstArgs& a, uint32_t t, double2* tile, uint32_t stile, int w,
                                                 int lane, uint64_t* wbar) {
  issue_contig_any_tile(a.x, tile_of<SIDE_CONTIG, false>(a, t), tile, stile, w, lane, wbar);
}

struct Lane {
  int f, q;
  double sq, cq;             // sin, cos of pi q / 512
  double2 w1, w8, w16, w24;  // W_512^{q}, ^{8q}, ^{16q}, ^{24q}
};

// opaque read-only loads: the lane constants are re-read (L1 hits) for every
// tile instead of living in registers across the tile loop; everything
// derived from them (32 sines, 31 twiddles) is loop-invariant, and a plain
// load would let the compiler hoist it all out of the loop and spill it
__device__ __forceinline__ double launder_d(double v) {
  double r;
  asm volatile("mov.b64 %0, %1;" : "=d"(r) : "d"(v));
  return r;
}

__device__ __forceinline__ double ld_opaque(const double* p) {
  double r;
  asm volatile("ld.global.nc.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_opaque2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}

__device__ __forceinline__ int launder_i(int v) {
  int r;
  asm volatile("mov.b32 %0, %1;" : "=r"(r) : "r"(v));
  return r;
}

// lane constants, re-derived per tile (lane index laundered: the smem
// offsets computed from q are loop-invariant too)
// (LAUNDER: the fused pass, whose larger live state otherwise spills the
// hoisted offsets; the plain passes are faster without)
template <bool LAUNDER = false>
__device__ __forceinline__ Lane lane_consts(const DstArgs& a, int lane_in) {
  Lane c;
  const int lane = LAUNDER ? launder_i(lane_in) : lane_in;
  c.f = lane >> 4;
  c.q = lane & 15;
  c.sq = ld_opaque(a.sn + c.q);
  c.cq = ld_opaque(a.sn + H - c.q);
  c.w1 = ld_opaque2(a.tw + c.q);
  c.w8 = ld_opaque2(a.tw + ((8 * c.q) & (N - 1)));
  c.w16 = ld_opaque2(a.tw + ((16 * c.q) & (N - 1)));
  c.w24 = ld_opaque2(a.tw + ((24 * c.q) & (N - 1)));
  return c;
}

// DST-I pre-processing of rows j and N - j into sc * y_j (m = row block,
// j = q + 16 m): the pass's output scale rides on the coefficients
// (s + 1/2) sc and (s - 1/2) sc, free next to the s +- 1/2 it replaces
__device__ __forceinline__ double2 pre_y(const Lane& c, int m, double2 xa, double2 xb, double sc, double hsc) {
  const double s = fma(c.sq, kc(m), c.cq * ks(m));  // sin(pi (q + 16 m) / 512)
  const double sp = fma(s, sc, hsc), sm = fma(s, sc, -hsc);
  double2 y = make_double2(fma(sp, xa.x, sm * xb.x), fma(sp, xa.y, sm * xb.y));
  if (m == 0 && c.q == 0) y = make_double2(0.0, 0.0);
  if (m == 16 && c.q == 0) y = make_double2((sc + sc) * xa.x, (sc + sc) * xa.y);
  return y;
}

// pre-processed input y_{q + 16 m} of FFT f of warp w
template <int RAW>
__device__ __forceinline__ void pre_read(const double2* tile, int w, const Lane& c_in, double2 (&v)[32], double sc,
                                         int sha = 0, int shb = 0, int sp = 512) {
  Lane c = c_in;
  const double hsc = 0.5 * sc;
  const int f = c.f, q = c.q, q7 = q & 7;
  // each batch's sines are computed from freshly laundered sin/cos, so the
  // compiler cannot precompute all 32 of them ahead of the loads
  auto batch = [&](int m) {
    if (m % PRE_BATCH == 0) {
      sched_fence();
      if (RAW != RAW_STRIDED) {  // (measured: the plain strided pass is faster without)
        c.sq = launder_d(c.sq);
        c.cq = launder_d(c.cq);
      }
    }
  };
  if constexpr (RAW == RAW_CONTIG) {
    // lines 4w + 2f (real) and 4w + 2f + 1 (imag), row j at j - 1 + shift
    // lines at 4w*512 + l*sp: sp = 512 (cp.async tiles, per-line shifts) or
    // the global pitch 511 / 512 (bulk-copied tiles, no shift)
    const double* d = reinterpret_cast<const double*>(tile) + 4 * w * 512 + 2 * f * sp;
    const double* ra = d + sha - 1;
    const double* rb = d + sp + shb - 1;
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      batch(m);
      const int j = (m == 0) ? (q == 0 ? 1 : q) : q + 16 * m;  // q + 16 m (row 0 -> any valid row)
      const int jp = 512 - q - 16 * m;                         // N - j (m = 0, q = 0: 512 -> clamp)
      const int jb = (m == 0 && q == 0) ? 1 : jp;
      v[m] = pre_y(c, m, make_double2(ra[j], rb[j]), make_double2(ra[jb], rb[jb]), sc, hsc);
    }
  } else if constexpr (RAW == RAW_STRIDED) {
    const int ch = 2 * w + f;
    const int la = tidx(q, ch);                                               // + 128 m
    const int lb = q == 0 ? 128 + ch : (16 - q) * 8 + (ch ^ ((8 - q7) & 7));  // + 128 (31 - m)
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      batch(m);
      const int ia = la + 128 * m;
      const int ib = (m == 0 && q == 0) ? la : lb + 128 * (31 - m);
      v[m] = pre_y(c, m, tile[ia], tile[ib], sc, hsc);
    }
  } else {
    // z layout in warp w's 16 KB of the tile
    const double2* zt = tile + 1024 * w;
    const int la = zidx(q, f);
    const int lb = q == 0 ? 32 + f : zidx(16 - q, f);
#pragma unroll
    for (int m = 0; m < 32; ++m) {
      batch(m);
      // bits 5..7 of the row: (m >> 1) for row q + 16 m, (31 - m) >> 1 for the
      // partner row (16 - q) + 16 (31 - m), (32 - m) >> 1 for q = 0 (row 16 (32 - m))
      const int ia = (la ^ ((m >> 1) & 7)) + 32 * m;
      int ib = q == 0 ? ((lb ^ (((32 - m) >> 1) & 7)) + 32 * (31 - m)) : ((lb ^ (((31 - m) >> 1) & 7)) + 32 * (31 - m));
      if (m == 0 && q == 0) ib = ia;
      v[m] = pre_y(c, m, zt[ia], zt[ib], sc, hsc);
    }
  }
}

// FFT of the pre-processed v (lane q of FFT f), split, scan, with the warp's
// 8 KB scratch.  On return ev[i] = S'_{2k}, od[i] = S'_{2k+1} for
// k = 16 q + i, S' = 2 * DST_raw (lines 2f / 2f+1 in .x / .y; ev[0] of lane
// 0 is S_0, unused).
#ifndef FL_REG_TWTAB
#define FL_REG_TWTAB 0
#endif
__device__ __forceinline__ void fft_split(double2* scr, const Lane& c, double2 (&v)[32], double2 (&ev)[16],
                                          double2 (&od)[16], const double2* twt = nullptr) {
  const int f = c.f, q = c.q, q7 = q & 7;
  double2* sf = scr + f * 256;
  dif<32>(v);
  // exchange in two rounds (k2 < 16, k2 >= 16): [k2'][q' ^ (k2' & 7)]
  // twiddles W_512^{q k2}, k2 = 8 h + l: W^{8qh} exact, then products by W^q
  double2 w0[16], w1[16];
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
        if (FL_REG_TWTAB) {
          // exact W_512^{q k2} from the CTA's table (k2-major, q fastest)
          if (k2) val = cmul(val, twt[k2 * 16 + q]);
        } else {
          if (h == 0 && l == 1) t = c.w1;
          if ((h == 0 && l >= 2) || (h > 0 && l >= 1)) t = cmul(t, c.w1);
          if (k2) val = cmul(val, t);
        }
        const int kk = k2 & 15;
        sf[kk * 16 + (q ^ (kk & 7))] = val;
      }
    }
    __syncwarp();
#pragma unroll
    for (int qq = 0; qq < 16; ++qq) {
      const double2 x = sf[q * 16 + (qq ^ q7)];
      if (rd == 0) w0[qq] = x; else w1[qq] = x;
    }
    __syncwarp();
  }
  dif<16>(w0);
  dif<16>(w1);
  // spectrum staging in two rounds: k < 256 (k1 < 8), then k >= 256; entry
  // kk = k mod 256 at kk ^ ((kk >> 4) & 7)
  double2 ck[16], cm[16];
#pragma unroll
  for (int rd = 0; rd < 2; ++rd) {
#pragma unroll
    for (int i = 0; i < 16; ++i) {
      const int k1 = brev(i, 4);
      if ((k1 >> 3) != rd) continue;
      const int k1l = k1 & 7;
      sf[32 * k1l + (q ^ ((2 * k1l) & 7))] = w0[i];
      sf[32 * k1l + 16 + (q ^ ((2 * k1l + 1) & 7))] = w1[i];
    }
    __syncwarp();
    if (rd == 0) {
#pragma unroll
      for (int i = 0; i < 16; ++i) ck[i] = sf[16 * q + (i ^ q7)];
    } else {
      // partner N - k of k = 16q + i: kk = 16 (15 - q) + (16 - i) for i >= 1,
      // 16 (16 - q) for i = 0 (q >= 1); k = 0 pairs with itself
#pragma unroll
      for (int i = 1; i < 16; ++i) cm[i] = sf[16 * (15 - q) + ((16 - i) ^ ((7 - q7) & 7))];
      cm[0] = q == 0 ? ck[0] : sf[16 * (16 - q) + ((16 - q) & 7)];
    }
    __syncwarp();
  }
  double2 run = make_double2(0.0, 0.0);
#pragma unroll
  for (int i = 0; i < 16; ++i) {
    double2 r = make_double2(ck[i].x + cm[i].x, ck[i].y + cm[i].y);
    ev[i] = make_double2(cm[i].y - ck[i].y, ck[i].x - cm[i].x);
    if (i == 0 && q == 0) r = ck[0];  // R_0 / 2 seeds S_1
    run.x += r.x;
    run.y += r.y;
    od[i] = run;
  }
  // exclusive offsets over the 16 lanes of this FFT
  double2 inc = run;
#pragma unroll
  for (int d = 1; d < 16; d <<= 1) {
    const double ux = __shfl_up_sync(0xffffffffu, inc.x, d, 16);
    const double uy = __shfl_up_sync(0xffffffffu, inc.y, d, 16);
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

// strided output, half hh (rows [256 hh, 256 hh + 256)): stage the lane's rows
// in its warp's scratch, then the CTA writes whole row segments.  Row
// r' = r0 + 16 s of the half (r0 = 4w + rho lane-constant) sits at
// sidx(r', f', w') = 32 s + (b ^ ((s >> 1) & 7)) with b lane-constant.
template <int SIDE_OUT>
__device__ __forceinline__ void store_strided(const DstArgs& a, uint32_t t, double2* scr_all, int w, int lane, int f,
                                              int q, const double2 (&ev)[16], const double2 (&od)[16], double sc) {
  const Tile tl = tile_of<SIDE_OUT, true>(a, t);
  double2* sw = scr_all + SCR * w;
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    // lane q holds rows [32 q, 32 q + 32): half hh is lanes q in [8 hh, 8 hh + 8)
    if ((q >> 3) == hh) {
      const int q7 = q & 7;
      double2* b = sw + 64 * q7;  // rows r' = 32 q7 + ..: sidx = 64 q7 + (zidx(r' & 31) ^ q7 ^ 2w)
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        const double2 e = make_double2(sc * ev[i].x, sc * ev[i].y);
        const double2 o = make_double2(sc * od[i].x, sc * od[i].y);
        if (i > 0 || q > 0) b[zidx(2 * i, f) ^ q7 ^ (2 * w)] = e;
        b[zidx(2 * i + 1, f) ^ q7 ^ (2 * w)] = o;
      }
    }
    __syncthreads();
    if (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 3) || a.scale == 12345.0) {
      if constexpr (SIDE_OUT == SIDE_VEC) {
        const int rho = lane >> 3, ch = lane & 7, fo = ch & 1, wo = ch >> 1;
        const int r0 = 4 * w + rho;  // rows r' = r0 + 16 s
        const double2* src = scr_all + SCR * wo;
        const int b = (2 * r0 + (fo ^ ((r0 >> 2) & 1))) ^ (2 * wo);
        const bool ok = 2 * ch < tl.lmax;
        const int64_t JS16 = 16 * tl.JS;
        double* y = a.y + tl.base + 2 * ch + (int64_t)(r0 + 256 * hh - 1) * tl.JS;
#pragma unroll
        for (int s = 0; s < 16; ++s) {
          const double2 val = src[32 * s + (b ^ ((s >> 1) & 7))];
          if (ok && (s > 0 || hh > 0 || r0 > 0)) *reinterpret_cast<double2*>(y) = val;
          y += JS16;
        }
      } else {
        const int rho = lane >> 4, cc = lane & 15, ch = cc >> 1, fo = ch & 1, wo = ch >> 1;
        const int r0 = 2 * w + rho;  // rows r' = r0 + 8 s
        const double* src = reinterpret_cast<const double*>(scr_all + SCR * wo) + (cc & 1);
        const int b = (2 * r0 + (fo ^ ((r0 >> 2) & 1))) ^ (2 * wo);  // r0 < 8: bits 5..7 of r' come from s
        const bool ok = cc < tl.lmax;
        const int64_t JS8 = 8 * tl.JS;
        double* y = a.y + tl.base + cc + (int64_t)(r0 + 256 * hh - 1) * tl.JS;
#pragma unroll
        for (int s = 0; s < 32; ++s) {
          // r' = r0 + 8 s: 2 r' = 2 r0 + 16 s, bit 2 of r' = bit 2 of r0 ^ bit 0 of s... (r0 < 8)
          const int rp_lo = (2 * r0 + 16 * (s & 1));  // 2 r' mod 32
          const int bb = (rp_lo + (fo ^ (((r0 + 8 * (s & 1)) >> 2) & 1))) ^ (2 * wo);
          const double val = src[2 * (32 * (s >> 1) + (bb ^ ((s >> 2) & 7)))];
          if (ok && (s > 0 || hh > 0 || r0 > 0)) *y = val;
          y += JS8;
        }
        (void)b;
      }
    }
    __syncthreads();
  }
}

// contiguous output of warp w (lines 4w .. 4w+3 of the tile) through its
// 8 KB scratch in two halves of positions p = r - 1: [0, 256) (rows 1 .. 256)
// and [256, 512) (rows 257 .. 511, position 511 is never stored).  Staging
// [line][256] with 16-byte chunks (positions 2c, 2c+1) at c ^ ((c >> 4) & 7):
// a lane writes (odd row, next even row) = (od[i], ev[i+1]) as one 16-byte
// store (8 active lanes of a quarter warp hit 8 chunk columns), the read-back
// is one 16-byte load per lane, 512 contiguous bytes per warp instruction,
// stored as 16 bytes where the line is 16-byte aligned.
__device__ __forceinline__ int cstg(int p) { return (((p >> 1) ^ ((p >> 5) & 7)) << 1) | (p & 1); }

__device__ __forceinline__ void store_contig_tile(const DstArgs& a, double* yout, const Tile& tl, double2* scr, int w,
                                                  int lane, int f, int q, const double2 (&ev)[16],
                                                  const double2 (&od)[16], double sc) {
  double* sd = reinterpret_cast<double*>(scr);
  double* la = sd + (2 * f) * 256;  // line 2f (.x), line 2f + 1 (.y) at + 256
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    if ((q >> 3) == hh) {
      // rows 32q + 2i + 1 and 32q + 2i + 2: positions pl = 32 (q - 8hh) + 2i (+1)
      const int base = 32 * (q - 8 * hh);
#pragma unroll
      for (int i = 0; i < 15; ++i) {
        const int pl = base + 2 * i;
        const int ph = cstg(pl);  // even
        *reinterpret_cast<double2*>(la + ph) = make_double2(sc * od[i].x, sc * ev[i + 1].x);
        *reinterpret_cast<double2*>(la + 256 + ph) = make_double2(sc * od[i].y, sc * ev[i + 1].y);
      }
      const int pl = base + 30;  // row 32q + 31 (od[15]); position + 1 belongs to the next lane
      la[cstg(pl)] = sc * od[15].x;
      la[256 + cstg(pl)] = sc * od[15].y;
    }
    // row 32q (ev[0], position 32q - 1) of lanes q in [8hh + 1, 8hh + 8]
    if (q >= 1 && ((q - 1) >> 3) == hh) {
      const int pl = 32 * q - 1 - 256 * hh;
      la[cstg(pl)] = sc * ev[0].x;
      la[256 + cstg(pl)] = sc * ev[0].y;
    }
    __syncwarp();
    if (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 3) || a.scale == 12345.0) {
#pragma unroll
      for (int l = 0; l < 4; ++l) {
        if (4 * w + l < tl.lmax) {
          const int64_t off = tl.base + (int64_t)(4 * w + l) * tl.LS + 256 * hh;  // element of position 256 hh
          const bool al = ((off & 1) == 0) && ((reinterpret_cast<uintptr_t>(yout) & 15) == 0);
          double* y = yout + off;
#pragma unroll
          for (int s = 0; s < 4; ++s) {
            const int c = lane + 32 * s;  // chunk: positions 2c, 2c + 1 of the half
            const double2 val = *reinterpret_cast<const double2*>(sd + l * 256 + 2 * (c ^ ((c >> 4) & 7)));
            const bool last = (hh == 1 && c == 127);  // position 511 is padding (or absent)
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
    }
    __syncwarp();
  }
}

__device__ __forceinline__ void store_contig(const DstArgs& a, uint32_t t, double2* scr, int w, int lane, int f,
                                             int q, const double2 (&ev)[16], const double2 (&od)[16], double sc) {
  store_contig_tile(a, a.y, tile_of<SIDE_CONTIG, true>(a, t), scr, w, lane, f, q, ev, od, sc);
}

// ---- TMA tensor stores of strided outputs ---------------------------------
// Lane q holds rows 32q .. 32q+31, i.e. global rows g = r - 1 = 32 qq + ii
// with (qq, ii) = (q, j - 1) for j = r - 32q >= 1 and (q - 1, 31) for j = 0.
// Staged as [ii][qq][16 columns] (the box of a 5-D tensor map {columns, qq
// (stride 32 rows), ii (stride 1 row), groups, outer}), rows written together
// (same ii, 8 consecutive qq) fall in 8 bank groups under the 128-byte
// swizzle.  Row 511 does not exist, so half 1 is two boxes: qq 8..14 x 32
// and qq 15 x 31 (three maps: A = qq 0..7, B, C).
struct OutMaps {
  CUtensorMap a, b, c;
};

__device__ __forceinline__ void tma_store_5d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3,
                                             int c4) {
  asm volatile("cp.async.bulk.tensor.5d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5, %6}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(c4)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_read() { asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory"); }
__device__ __forceinline__ void bulk_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }

// double2 index of (qq, ii, chunk) in the staging of half hh
__device__ __forceinline__ int stg_tma_idx(int hh, int qq, int ii, int ch) {
  if (hh == 0) {
    const int R = ii * 8 + qq;
    return R * 8 + (ch ^ (R & 7));
  }
  if (qq < 15) {
    const int R = ii * 7 + (qq - 8);
    return R * 8 + (ch ^ (R & 7));
  }
  return 1792 + ii * 8 + (ch ^ (ii & 7));
}

// DEFER: half 1's staging is drained by the kernel before the next exchange
// instead of here (measured: helps the fused pass, costs the plain one)
template <bool DEFER>
__device__ __forceinline__ void store_strided_tma_at(const OutMaps* maps, int c0, uint32_t g, uint32_t o, double2* stg,
                                                     int w, int f, int q, const double2 (&ev)[16],
                                                     const double2 (&od)[16]) {
  const int ch = 2 * w + f;
  // the staging interleaves all four warps' columns over the whole 32 KB of
  // scratch: every warp must be done with its exchange/spectrum first
  __syncthreads();
#pragma unroll 1
  for (int hh = 0; hh < 2; ++hh) {
    if ((q >> 3) == hh) {
#pragma unroll
      for (int i = 0; i < 16; ++i) {
        if (i > 0) stg[stg_tma_idx(hh, q, 2 * i - 1, ch)] = ev[i];  // j = 2i
        stg[stg_tma_idx(hh, q, 2 * i, ch)] = od[i];                 // j = 2i + 1
      }
    }
    if (q >= 1 && ((q - 1) >> 3) == hh) stg[stg_tma_idx(hh, q - 1, 31, ch)] = ev[0];  // j = 0
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0 && !(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 3)) {
      if (hh == 0) {
        tma_store_5d(&maps->a, stg, c0, 0, 0, (int)g, (int)o);
      } else {
        tma_store_5d(&maps->b, stg, c0, 8, 0, (int)g, (int)o);
        tma_store_5d(&maps->c, stg + 1792, c0, 15, 0, (int)g, (int)o);
      }
      bulk_commit();
      if (!DEFER || hh == 0) bulk_wait_read();
    }
    if (!DEFER || hh == 0) __syncthreads();
  }
}

template <bool DEFER>
__device__ __forceinline__ void store_strided_tma(const DstArgs& a, const OutMaps* maps, uint32_t t, double2* stg,
                                                  int w, int f, int q, const double2 (&ev)[16],
                                                  const double2 (&od)[16]) {
  const uint32_t o = a.div_blk.div(t);
  const uint32_t rr = t - o * a.div_blk.d;
  const uint32_t g = a.div_chunk.div(rr);
  const int c0 = (int)(rr - g * a.div_chunk.d) * 16;
  store_strided_tma_at<DEFER>(maps, c0, g, o, stg, w, f, q, ev, od);
}

// TMA load of strided tile t: two 256-row boxes of 16 columns, rows -1 ..
// 254 (row -1 out of range: zeros) and 255 .. 510 into tile rows 0 .. 511;
// the 128-byte swizzle is exactly tidx's chunk ^ (row & 7)
__device__ __forceinline__ void tma_issue_at(const CUtensorMap* map, int c0, int g, int o, double2* tile,
                                             uint64_t* bar) {
  mbar_expect_tx(bar, (uint32_t)(TILE * sizeof(double2)));
  tma_load_4d(tile, map, c0, -1, g, o, bar);
  tma_load_4d(tile + TILE / 2, map, c0, 255, g, o, bar);
}
__device__ __forceinline__ void tma_issue_grp(const DstArgs& a, const CUtensorMap* map, uint32_t t, double2* tile,
                                              uint64_t* bar) {
  const uint32_t o = a.div_blk.div(t);
  const uint32_t r = t - o * a.div_blk.d;
  const uint32_t g = a.div_chunk.div(r);
  const int c0 = (int)(r - g * a.div_chunk.d) * 16;
  tma_issue_at(map, c0, (int)g, (int)o, tile, bar);
}

// Persistent CTAs of 4 warps (one 16-line tile at a time), 2 per SM.
// Strided sides: CTA-cooperative tiles (TMA: TMA loads; TST: TMA stores);
// contiguous sides: warp-local lines.  MID: forward, core (lane-ordered,
// full.lane_core / line_lane_core), inverse in one pass.
template <int SIDE_IN, int SIDE_OUT, bool MID, bool TMA, bool TST>
__global__ void __launch_bounds__(32 * NWARP, 2) k_dst_grp(const DstArgs a, const __grid_constant__ CUtensorMap map,
                                                           const __grid_constant__ OutMaps omaps) {
  extern __shared__ __align__(1024) double2 smem_grp[];
  double2* const tile = smem_grp;
  double2* const scr_all = smem_grp + TILE;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(scr_all + NWARP * SCR);
  uint64_t* const wbar = bar + 1 + (threadIdx.x >> 5);  // per-warp barrier of bulk line copies
  double2* const twt = scr_all + NWARP * SCR + 4;        // FL_REG_TWTAB: W_512^{q k2}, [k2][q]
  if (FL_REG_TWTAB) {
    for (int i = threadIdx.x; i < 512; i += 32 * NWARP) twt[i] = __ldg(&a.tw[((i & 15) * (i >> 4)) & (N - 1)]);
    __syncthreads();
  }
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const scr = scr_all + SCR * w;
  const uint32_t stile = smem_u32(tile);
  const uint32_t ntiles = (uint32_t)a.ntiles;
  uint32_t t = blockIdx.x;
  constexpr bool STRIDED = SIDE_IN != SIDE_CONTIG;
  static_assert(!TMA || SIDE_IN == SIDE_VEC, "TMA tiles need 16-byte aligned strided input");
  static_assert(!TST || SIDE_OUT == SIDE_VEC, "TMA stores need 16-byte aligned strided output");
  uint32_t phase = 0;
  auto issue_next = [&](uint32_t tt) {
    if constexpr (TMA) {
      if (threadIdx.x == 0 && !(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) tma_issue_grp(a, &map, tt, tile, bar);
    } else if constexpr (STRIDED) {
      issue_strided<SIDE_IN>(a, tt, stile, w, lane);
    } else {
      issue_contig_any(a, tt, tile, stile, w, lane, wbar);
    }
  };
  uint32_t wphase = 0;
  if constexpr (!STRIDED || MID) {
    if (lane == 0) {
      mbar_init(wbar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncwarp();
  }
  if constexpr (TMA) {
    if ((stile & 1023u) != 0) __trap();  // the 128-byte swizzle needs a 1024-byte aligned tile
    if (threadIdx.x == 0) {
      mbar_init(bar, 1);
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
  }
  if (t < ntiles) issue_next(t);
  cp_commit();
  for (; t < ntiles; t += gridDim.x) {
    const uint32_t tn = t + gridDim.x;
    if constexpr (TMA) {
      if (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) mbar_wait(bar, phase);
      phase ^= 1;
    }
    int sha = 0, shb = 0, sp = 512;  // contiguous tiles: line shifts and smem line pitch
    if constexpr (!STRIDED) {
      const Tile tin = tile_of<SIDE_CONTIG, false>(a, t);
      if (contig_bulk(a, tin, w)) {
        if (!(FL_REG_NOMEM == 1 || FL_REG_NOMEM == 2)) mbar_wait(wbar, wphase);
        wphase ^= 1;
        sp = (int)tin.LS;
      } else {
        sha = line_shift(tin, 4 * w + 2 * (lane >> 4));
        shb = line_shift(tin, 4 * w + 2 * (lane >> 4) + 1);
      }
    }
    cp_wait<0>();
    // TMA tiles: every thread waited on the tile's mbarrier itself, which
    // makes the bytes visible to it; only cooperative cp.async tiles need the
    // CTA barrier
    if constexpr (STRIDED && !TMA) __syncthreads();
    if constexpr (!STRIDED) __syncwarp();
    double2 v[32], ev[16], od[16];
    if constexpr (!MID) {
      const Lane c = lane_consts(a, lane);
      pre_read<STRIDED ? RAW_STRIDED : RAW_CONTIG>(tile, w, c, v, 0.5 * a.scale, sha, shb, sp);
      // the tile's generic-proxy reads must be ordered before the async-proxy
      // refill (TMA / bulk copy / cp.async into the same bytes): bar.sync
      // alone orders only the generic proxy
      proxy_fence_async();
      if (STRIDED) __syncthreads(); else __syncwarp();
      if (tn < ntiles) issue_next(tn);
      cp_commit();
      fft_split(scr, c, v, ev, od, twt);
    } else {
      // forward, core, inverse: a rolled loop keeps one copy of the FFT code
      // (two inlined copies do not fit the register file)
#pragma unroll 1
      for (int ph = 0; ph < 2; ++ph) {
        // v is (re)defined at the top of both phases, so it is dead across
        // the back edge
        if (ph == 0) {
          pre_read<STRIDED ? RAW_STRIDED : RAW_CONTIG>(tile, w, lane_consts<true>(a, lane), v, 0.25 * a.scale, sha,
                                                       shb, sp);
        } else {
          pre_read<RAW_Z>(tile, w, lane_consts<true>(a, lane), v, 1.0);
        }
        // phase 0: the tile is consumed, quarter w (16 KB) is the warp's own
        // from here; phase 1: every warp has read its z, the tile is free.
        // Either way the next writes into these bytes come from the async
        // proxy (core slice / TMA / bulk refill): fence the generic-proxy
        // reads (and phase 1's z writes) first
        proxy_fence_async();
        if (TST && ph == 0 && threadIdx.x == 0) bulk_wait_read();  // previous tile's half-1 store
        if (STRIDED) __syncthreads(); else __syncwarp();
        if (ph == 0) {
          // bring the unit's lane-ordered core slice into quarter w while the
          // forward FFT runs
          // (one bulk copy: the slice is 16 KB contiguous in lane order)
          if (lane == 0 && !FL_REG_NOMEM) {
            mbar_expect_tx(wbar, 16384u);
            bulk_load(tile + 1024 * w, reinterpret_cast<const double2*>(a.core) + (size_t)(4 * t + w) * 1024, 16384u,
                      wbar);
          }
        } else {
          if (tn < ntiles) issue_next(tn);
          cp_commit();
        }
        // shared addressing survives: the laundered part is an integer offset
        fft_split(scr_all + launder_i(SCR * w), lane_consts<true>(a, lane), v, ev, od, twt);
        if (ph == 0) {
          // z = S' .* core for rows 2k, 2k+1 (k = 16 q + i): multiply in
          // registers (core entry (i', lane) at 32 i' + lane), then write z
          // over the core in the z layout
          if (!FL_REG_NOMEM) mbar_wait(wbar, wphase);
          wphase ^= 1;
          __syncwarp();
          const double2* cw = tile + 1024 * w + lane;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            const double2 ce = cw[32 * (2 * i)], co = cw[32 * (2 * i + 1)];
            ev[i] = make_double2(ev[i].x * ce.x, ev[i].y * ce.y);
            od[i] = make_double2(od[i].x * co.x, od[i].y * co.y);
          }
          __syncwarp();
          const int q = lane & 15, f = lane >> 4, q7 = q & 7;
          double2* zt = tile + 1024 * w + 64 * q;
#pragma unroll
          for (int i = 0; i < 16; ++i) {
            if (i > 0 || q > 0) zt[zidx(2 * i, f) ^ q7] = ev[i];
            zt[zidx(2 * i + 1, f) ^ q7] = od[i];
          }
          __syncwarp();
        }
      }
    }
    // the scale (0.5 per split, nrm, alpha) was applied in the first pre-processing
    const double sc = 1.0;
    if constexpr (STRIDED) {
      if constexpr (TST) {
        store_strided_tma<MID>(a, &omaps, t, scr_all, w, lane >> 4, lane & 15, ev, od);
      } else {
        store_strided<SIDE_OUT>(a, t, scr_all, w, lane, lane >> 4, lane & 15, ev, od, sc);
      }
    } else {
      store_contig(a, t, scr, w, lane, lane >> 4, lane & 15, ev, od, sc);
    }
  }
  cp_wait<0>();
  if (TST && threadIdx.x == 0) bulk_wait_all();
}

constexpr size_t grp_smem_bytes() {
  return (size_t)(TILE + NWARP * SCR + 4 + (FL_REG_TWTAB ? 512 : 0)) * sizeof(double2);
}

}  // namespace rg
}  // namespace fl
