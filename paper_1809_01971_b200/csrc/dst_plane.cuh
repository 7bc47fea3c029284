// Plane-fused DST-I passes for the 511^3 apply (configs[2]): the last mode
// and mode 1 of one i0-plane in ONE persistent kernel, the intermediate plane
// held in an L2-resident ring instead of a full-size HBM tensor.
//
// The 5-pass apply (fl_apply_full_lanes) moves 16 B/DoF per plain pass; the
// pair "last mode, then mode 1" writes a 1.07 GB intermediate and reads it
// back.  A 511 x 512 plane is only 2.09 MB, so here the first pass writes
// each plane into one of 16 ring slots (33.5 MB, stays in the 126 MB L2;
// slot = plane mod 16) and the second pass reads it from there: 16 B/DoF of
// DRAM traffic for the two transforms instead of 32.  Forward direction:
//   A items: 16-line tiles of the last mode, dense x (pitch 511) -> ring
//            (pitch 512, padding written as 0), per-warp bulk loads;
//   B items: 16-column tiles of mode 1 on a ring plane -> work tensor
//            (padded layout), TMA tile loads and TMA tensor stores.
// Inverse direction (after the fused mode-0 pass):
//   A items: mode 1 on a work plane -> ring (TMA loads, TMA stores);
//   B items: last mode, ring -> dense y (pitch 511), per-warp bulk loads.
// The ring is addressed by global line L = 511 i0 + i1 as L mod (16 * 511):
// 8176 is a multiple of 16, so a 16-line tile never wraps.
//
// Scheduling: items are dealt by a global ticket counter in a fixed order,
// round r = [A items starting in plane r, B items of plane r - LAG], and
// every dependency points to an earlier ticket:
//   B(p) needs all A tiles covering plane p       (ready[p] counter),
//   A(p) may overwrite slot p mod 16 only after all B items of plane p - 16
//   have read it                                  (consumed[p - 16]).
// A CTA holds its current item, the next one (loads issued early, or
// deferred when its producers are not done yet) and one dealt-ahead ticket.
// Completion signals of finished items are published before any wait and a
// wait only ever targets earlier tickets, so the smallest unfinished ticket
// is always some CTA's current item and can progress: deadlock-free without
// any co-residency assumption (non-resident CTAs hold no tickets).
// Completion of generic-proxy stores is published by __threadfence + a
// release atomic; of TMA stores by cp.async.bulk.wait_group 0 + a proxy
// fence first.  Consumers acquire, then fence the async proxy before their
// TMA / bulk loads read the ring.
#pragma once

#include "dst_reg.cuh"

namespace fl {
namespace pl {

using namespace rg;

constexpr int NP = 511;             // planes (i0), lines per plane (i1), line length (i2)
constexpr int PITCH = 512;          // padded line pitch of the ring and the work tensor
constexpr int SLOTS = 16;           // ring slots
constexpr int RING_LINES = SLOTS * NP;  // 8176 = 511 tiles of 16 lines
constexpr int LINES = NP * NP;      // 261121 lines of the last mode
constexpr int ATILES = (LINES + 15) / 16;  // 16321 tiles of 16 lines
constexpr int BITEMS = 32;          // 16-column tiles per plane (512 columns)
#ifndef FL_PLANE_LAG
#define FL_PLANE_LAG 2
#endif
constexpr int LAG = FL_PLANE_LAG;
constexpr int ROUNDS = NP + LAG;

struct PlaneArgs {
  DstArgs a;           // tw / sn tables (lane constants)
  const double* x;     // forward: dense x; inverse: work tensor
  double* y;           // forward: work tensor; inverse: dense y
  double* ring;        // SLOTS x 511 x 512
  int* ready;          // [NP] producer completions per plane
  int* consumed;       // [NP] consumer reads per plane
  unsigned* ticket;    // global ticket counter
  double scale_a, scale_b;  // output scales of the A and B transforms (incl. the DST normalisation)
};

// 16-line tiles (global line tiles) touching plane p: their count
__host__ __device__ constexpr int tiles_touching(int p) { return (NP * p + NP - 1) / 16 - (NP * p) / 16 + 1; }
// first line tile whose first line lies in plane r (r <= NP)
__host__ __device__ constexpr int first_tile_of_round(int r) { return (NP * r + 15) / 16; }

// tickets dealt before round r
__device__ __forceinline__ int tickets_before(int r, bool fwd) {
  const int rr = r < NP ? r : NP;
  int d = r - LAG;
  d = d < 0 ? 0 : (d > NP ? NP : d);
  // forward: line tiles of rounds < r, then B items of planes < r - LAG;
  // inverse: plane items (32 each) of rounds < r, then line tiles of planes < r - LAG
  return fwd ? first_tile_of_round(rr) + BITEMS * d : BITEMS * rr + first_tile_of_round(d);
}

struct Item {
  int kind;   // 0: none (past the end), 1: line tile (last mode), 2: plane chunk (mode 1)
  int idx;    // line tile t, or plane p
  int chunk;  // plane chunk c (kind 2)
};

__device__ __forceinline__ Item decode(unsigned k, bool fwd) {
  Item it{0, 0, 0};
  const int total = tickets_before(ROUNDS, fwd);
  if ((int)k >= total) return it;
  int r = (int)((long long)k * 16 / 1023);  // ~63.94 tickets per round
  if (r > ROUNDS - 1) r = ROUNDS - 1;
  while (r > 0 && tickets_before(r, fwd) > (int)k) --r;
  while (r < ROUNDS - 1 && tickets_before(r + 1, fwd) <= (int)k) ++r;
  const int off = (int)k - tickets_before(r, fwd);
  const int rr = r < NP ? r : NP;
  if (fwd) {
    const int na = (r < NP) ? first_tile_of_round(rr + 1) - first_tile_of_round(rr) : 0;
    if (off < na) {
      it.kind = 1;
      it.idx = first_tile_of_round(rr) + off;
    } else {
      it.kind = 2;
      it.idx = r - LAG;
      it.chunk = off - na;
    }
  } else {
    const int na = (r < NP) ? BITEMS : 0;
    if (off < na) {
      it.kind = 2;
      it.idx = r;
      it.chunk = off;
    } else {
      it.kind = 1;
      it.idx = first_tile_of_round(r - LAG) + (off - na);
    }
  }
  return it;
}

__device__ __forceinline__ int ld_acquire(const int* p) {
  int v;
  asm volatile("ld.acquire.gpu.global.b32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_add(int* p, int v) {
  asm volatile("red.release.gpu.global.add.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void fence_proxy_async_global() { asm volatile("fence.proxy.async.global;" ::: "memory"); }

__device__ __forceinline__ void spin_until(const int* p, int target) {
  if (ld_acquire(p) >= target) return;
  while (ld_acquire(p) < target) __nanosleep(64);
}

// line tile t: planes of its first and last line
__device__ __forceinline__ void tile_planes(int t, int& plo, int& phi, int& lmax) {
  const int L0 = 16 * t;
  lmax = LINES - L0 < 16 ? LINES - L0 : 16;
  plo = L0 / NP;
  phi = (L0 + lmax - 1) / NP;
}

// producers that must have finished before line tile t may be loaded (inverse)
// / plane-chunk items of plane p may be loaded (forward); true when met now
__device__ __forceinline__ bool deps_met(const PlaneArgs& P, const Item& it, bool fwd) {
  if (it.kind == 0) return true;
  if (fwd) {
    if (it.kind != 2) return true;  // line tiles read x
    return ld_acquire(P.ready + it.idx) >= tiles_touching(it.idx);
  }
  if (it.kind != 1) return true;  // plane chunks read the work tensor
  int plo, phi, lmax;
  tile_planes(it.idx, plo, phi, lmax);
  return ld_acquire(P.ready + plo) >= BITEMS && ld_acquire(P.ready + phi) >= BITEMS;
}

__device__ __forceinline__ void wait_deps(const PlaneArgs& P, const Item& it, bool fwd) {
  if (it.kind == 0) return;
  if (fwd) {
    if (it.kind == 2) spin_until(P.ready + it.idx, tiles_touching(it.idx));
    return;
  }
  if (it.kind == 1) {
    int plo, phi, lmax;
    tile_planes(it.idx, plo, phi, lmax);
    spin_until(P.ready + plo, BITEMS);
    spin_until(P.ready + phi, BITEMS);
  }
}

// ring side of a line tile (pitch 512) and its dense side (pitch 511)
__device__ __forceinline__ Tile ring_tile(int t, int lmax) {
  Tile r;
  r.base = (int64_t)((16 * t) % RING_LINES) * PITCH;
  r.JS = 1;
  r.LS = PITCH;
  r.lmax = lmax;
  return r;
}
__device__ __forceinline__ Tile dense_tile(int t, int lmax) {
  Tile r;
  r.base = (int64_t)(16 * t) * NP;
  r.JS = 1;
  r.LS = NP;
  r.lmax = lmax;
  return r;
}

// FWD: forward direction (dense x -> ring -> work), else inverse.
// mapL: TMA load map of the plane-chunk side (forward: the ring, outer =
// slot; inverse: the work tensor, outer = plane); mapsS: TMA store maps of
// the plane-chunk output (forward: work, outer = plane; inverse: ring).
//
// Per item: [top: publish the previous producer item (thread 0: TMA-store
// completion; all: __threadfence) | thread 0 reads the next ticket (dealt
// one round earlier), checks whether its producers are done, deals the
// ticket after it | wait for the current data | pre-processing out of the
// tile | CTA barrier | release atomics, consumer signal | issue the next
// item's loads (or defer them) | FFT | store].  Ticket slots are
// triple-buffered in shared memory: slot i % 3 is written by thread 0 at
// the top of iteration i - 1 and read by everyone after iteration i's
// barrier, and its next write (top of i + 2) comes after barrier i + 1.
template <bool FWD>
__global__ void __launch_bounds__(32 * NWARP, 2) k_plane(const PlaneArgs P, const __grid_constant__ CUtensorMap mapL,
                                                        const __grid_constant__ OutMaps mapsS) {
  extern __shared__ __align__(1024) double2 smem_pl[];
  double2* const tile = smem_pl;
  double2* const scr_all = smem_pl + TILE;
  uint64_t* const bar = reinterpret_cast<uint64_t*>(scr_all + NWARP * SCR);
  uint64_t* const wbar = bar + 1 + (threadIdx.x >> 5);
  unsigned* const s_tk = reinterpret_cast<unsigned*>(bar + 1 + NWARP);  // [0..2] tickets, [3..5] deps met, [6] current
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  double2* const scr = scr_all + SCR * w;
  const uint32_t stile = smem_u32(tile);
  const DstArgs& a = P.a;
  if ((stile & 1023u) != 0) __trap();
  if (lane == 0) mbar_init(wbar, 1);
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    s_tk[6] = atomicAdd(P.ticket, 1u);
  }
  __syncthreads();
  uint32_t phase = 0, wphase = 0;

  // issue the loads of item `it` into the tile buffer (the caller made sure
  // the buffer is free and the producers are done)
  auto issue = [&](const Item& it) {
    if (it.kind == 0) return;
    if (it.kind == 1) {
      int plo, phi, lmax;
      tile_planes(it.idx, plo, phi, lmax);
      const Tile tl = FWD ? dense_tile(it.idx, lmax) : ring_tile(it.idx, lmax);
      if (!FWD && lane == 0) fence_proxy_async_global();  // ring written by other CTAs' TMA stores
      issue_contig_any_tile(FWD ? P.x : P.ring, tl, tile, stile, w, lane, wbar);
    } else if (threadIdx.x == 0) {
      if (FWD) fence_proxy_async_global();  // ring written by other CTAs' generic stores
      tma_issue_at(&mapL, 16 * it.chunk, 0, FWD ? it.idx % SLOTS : it.idx, tile, bar);
    }
    cp_commit();
  };

  Item cur = decode(s_tk[6], FWD);
  __syncthreads();
  if (threadIdx.x == 0) {
    wait_deps(P, cur, FWD);  // nothing held yet: blocking is safe
    if (cur.kind != 0) s_tk[0] = atomicAdd(P.ticket, 1u);
  }
  __syncthreads();
  issue(cur);
  bool deferred = false;
  // completion signal of the previous producer item, published in the next
  int pend_kind = 0, pend_a = -1, pend_b = -1;
  auto publish = [&]() {
    if (threadIdx.x == 0) {
      red_release_add(P.ready + pend_a, 1);
      if (pend_b >= 0) red_release_add(P.ready + pend_b, 1);
    }
    pend_kind = 0;
  };

  for (int it = 0; cur.kind != 0; ++it) {
    const int sl = it % 3, sn = (it + 1) % 3;
    if (pend_kind) {
      if (pend_kind == 2 && threadIdx.x == 0) {
        bulk_wait_all();  // this CTA's TMA stores into the ring are complete
        fence_proxy_async_global();
      }
      __threadfence();
    }
    if (deferred) {
      // publish first, then wait for the producers (this CTA holds no other
      // unfinished item now), then load
      __syncthreads();
      if (pend_kind) publish();
      if (threadIdx.x == 0) wait_deps(P, cur, FWD);
      __syncthreads();
      issue(cur);
      deferred = false;
    }
    if (threadIdx.x == 0) {
      const Item nx = decode(s_tk[sl], FWD);
      s_tk[3 + sl] = deps_met(P, nx, FWD) ? 1u : 0u;
      if (nx.kind != 0) s_tk[sn] = atomicAdd(P.ticket, 1u);
    }
    const bool lines = cur.kind == 1;
    int plo = 0, phi = 0, lmax = 16;
    if (lines) tile_planes(cur.idx, plo, phi, lmax);
    // ---- wait for the current item's data ---------------------------------
    int sha = 0, shb = 0, sp = 512;
    if (lines) {
      const Tile tin = FWD ? dense_tile(cur.idx, lmax) : ring_tile(cur.idx, lmax);
      if (contig_bulk_p(FWD ? P.x : P.ring, tin, w)) {
        mbar_wait(wbar, wphase);
        wphase ^= 1;
        sp = (int)tin.LS;
      } else {
        sha = line_shift(tin, 4 * w + 2 * (lane >> 4));
        shb = line_shift(tin, 4 * w + 2 * (lane >> 4) + 1);
      }
      cp_wait<0>();
      __syncwarp();
    } else {
      mbar_wait(bar, phase);
      phase ^= 1;
    }
    // ---- pre-processing out of the tile; then the tile is free -------------
    double2 v[32], ev[16], od[16];
    const Lane c = lane_consts(a, lane);
    const double sc = 0.5 * ((lines == FWD) ? P.scale_a : P.scale_b);
    if (lines)
      pre_read<RAW_CONTIG>(tile, w, c, v, sc, sha, shb, sp);
    else
      pre_read<RAW_STRIDED>(tile, w, c, v, sc);
    proxy_fence_async();
    __syncthreads();
    if (pend_kind) publish();
    // a consumer item's ring data is in registers now
    if (threadIdx.x == 0) {
      if (FWD && !lines) red_release_add(P.consumed + cur.idx, 1);
      if (!FWD && lines) {
        red_release_add(P.consumed + plo, 1);
        if (phi != plo) red_release_add(P.consumed + phi, 1);
      }
    }
    const Item nxt = decode(s_tk[sl], FWD);
    if (s_tk[3 + sl])
      issue(nxt);
    else
      deferred = true;
    fft_split(scr, c, v, ev, od, nullptr);
    // ---- store -------------------------------------------------------------
    if (lines) {
      if (FWD) {
        // the ring slots of planes plo, phi: their previous planes must be read
        if (lane == 0) {
          if (plo >= SLOTS) spin_until(P.consumed + plo - SLOTS, BITEMS);
          if (phi != plo && phi >= SLOTS) spin_until(P.consumed + phi - SLOTS, BITEMS);
        }
        __syncwarp();
        store_contig_tile(a, P.ring, ring_tile(cur.idx, lmax), scr, w, lane, lane >> 4, lane & 15, ev, od, 1.0);
        pend_kind = 1;
        pend_a = plo;
        pend_b = (phi != plo) ? phi : -1;
      } else {
        store_contig_tile(a, P.y, dense_tile(cur.idx, lmax), scr, w, lane, lane >> 4, lane & 15, ev, od, 1.0);
      }
    } else {
      if (!FWD && cur.idx >= SLOTS && threadIdx.x == 0) {
        spin_until(P.consumed + cur.idx - SLOTS, tiles_touching(cur.idx - SLOTS));
        fence_proxy_async_global();
      }
      // (store_strided_tma_at starts with a CTA barrier)
      store_strided_tma_at<false>(&mapsS, 16 * cur.chunk, 0, FWD ? cur.idx : cur.idx % SLOTS, scr_all, w,
                                  lane >> 4, lane & 15, ev, od);
      if (!FWD) {
        pend_kind = 2;
        pend_a = cur.idx;
        pend_b = -1;
      }
    }
    cur = nxt;
  }
  // the last producer item
  if (pend_kind) {
    if (pend_kind == 2 && threadIdx.x == 0) {
      bulk_wait_all();
      fence_proxy_async_global();
    }
    __threadfence();
    __syncthreads();
    publish();
  }
  cp_wait<0>();
  if (threadIdx.x == 0) bulk_wait_all();
}

constexpr size_t plane_smem_bytes() { return (size_t)(TILE + NWARP * SCR + 8) * sizeof(double2); }

}  // namespace pl
}  // namespace fl
