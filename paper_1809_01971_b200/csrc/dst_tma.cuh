// TMA-fed variant of the strided DST pass (see dst_fft.cuh for the FFT).
//
// On strided tiles the raw tile (rows j of 2*NFFT consecutive columns) has
// exactly the shared-memory cell layout: row j holds cell position j+1, one
// complex cell per line pair.  So the Tensor Memory Accelerator can copy
// the next tile straight into a second cell buffer while the current tile
// is transformed: one thread issues cp.async.bulk.tensor boxes (2*NFFT
// columns x BR rows, out-of-bounds rows/columns zero-filled) that complete
// on an mbarrier; the DST-I pre-processing then runs in place in shared
// memory (rows j and N-j of a line pair are combined where they lie).
// NBUF = 2: one CTA per SM with two cell buffers; NBUF = 1: two CTAs per SM.
// Opt-in (FL_TMA=1|2): measured at n=511 (mode-1 pass) 0.650 / 0.653 ms vs
// 0.624 ms for the LDG kernel of dst_fft.cuh — the in-place pre-processing
// pass costs more shared-memory bandwidth than the hidden load latency
// saves on this shared-memory-bound transform.
#pragma once

#include <cuda.h>

#include "dst_fft.cuh"

namespace fl {

struct TmaGeom {
  int box_rows;    // rows per TMA box (<= 256)
  int nbox;        // boxes per tile
  int delta;       // buffer row of position 1 (TMA destination, 128-byte aligned)
  int rows_total;  // rows per cell buffer
  uint32_t tx_bytes;  // bytes per tile (all boxes, zero fill included)
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, int c0, int c1, int c2, int c3,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3, %4, %5}], [%6];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(c3), "r"(smem_u32(bar))
      : "memory");
}

// copy tile `tile` (strided: block o, group g, first column c0) into buf
template <int NFFT>
__device__ __forceinline__ void tma_issue_tile(const DstArgs& a, const CUtensorMap* map, const TmaGeom& geo,
                                               int64_t tile, double2* buf, uint64_t* bar) {
  constexpr int C = 2 * NFFT;
  const uint32_t t32 = (uint32_t)tile;
  const uint32_t o = a.div_blk.div(t32);
  const uint32_t r = t32 - o * a.div_blk.d;
  const uint32_t g = a.div_chunk.div(r);
  const int c0 = (int)(r - g * a.div_chunk.d) * C;
  mbar_expect_tx(bar, geo.tx_bytes);
  for (int b = 0; b < geo.nbox; ++b)
    tma_load_4d(buf + (size_t)(geo.delta + b * geo.box_rows) * NFFT, map, c0, b * geo.box_rows, (int)g, (int)o, bar);
}

// DST-I pre-processing in place: item (u, k) combines rows j = k+1 and N-j
template <int LOGN, int NFFT, int NT>
__device__ __forceinline__ void dst_pre_inplace(const DstArgs& a, const Cells<LOGN, NFFT, false>& cs) {
  using SP = Split<LOGN, NFFT, NT, false>;
  constexpr int N = SP::N, H = SP::H, PER = SP::PER;
  int k0, u0;
  SP::base(threadIdx.x, k0, u0);
  double2 va[PER], vb[PER];
#pragma unroll
  for (int it = 0; it < PER; ++it) {
    const int j = k0 + SP::MS(it) + 1;
    va[it] = make_double2(0.0, 0.0);
    vb[it] = make_double2(0.0, 0.0);
    if (SP::ok(threadIdx.x, it)) {
      va[it] = cs.ld(j, u0);
      if (j < H) vb[it] = cs.ld(N - j, u0);
    }
  }
#pragma unroll
  for (int it = 0; it < PER; ++it)
    if (SP::ok(threadIdx.x, it)) pre_pair(cs, a.sn, u0, k0 + SP::MS(it) + 1, va[it], vb[it]);
  for (int u = threadIdx.x; u < NFFT; u += NT) cs.st(0, u, make_double2(0.0, 0.0));
}

// NBUF = 2: one CTA per SM, the next tile lands while this one computes.
// NBUF = 1: two CTAs per SM (64 registers), the refill of one CTA's buffer
// overlaps the other CTA's compute.
template <int LOGN, int NFFT, int NT, bool TW3, int NBUF>
__global__ void __launch_bounds__(NT, 3 - NBUF) k_dst_tma(const DstArgs a, const __grid_constant__ CUtensorMap map,
                                                        const TmaGeom geo) {
  using CS = Cells<LOGN, NFFT, false>;
  constexpr int C = 2 * NFFT;
  extern __shared__ __align__(128) unsigned char smem_tma[];
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(smem_tma) + 127) & ~uintptr_t(127));
  const size_t buf_bytes = (size_t)geo.rows_total * NFFT * sizeof(double2);
  double2* buf0 = reinterpret_cast<double2*>(base);
  double2* buf1 = reinterpret_cast<double2*>(base + (NBUF - 1) * buf_bytes);
  double2* scr = reinterpret_cast<double2*>(base + NBUF * buf_bytes);
  uint64_t* bar = reinterpret_cast<uint64_t*>(scr + NFFT * (NT / 32));
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    if (blockIdx.x < a.ntiles) tma_issue_tile<NFFT>(a, &map, geo, blockIdx.x, buf0, &bar[0]);
    if (NBUF == 2 && blockIdx.x + gridDim.x < a.ntiles)
      tma_issue_tile<NFFT>(a, &map, geo, blockIdx.x + gridDim.x, buf1, &bar[1]);
  }
  int i = 0;
  for (int64_t tile = blockIdx.x; tile < a.ntiles; tile += gridDim.x, ++i) {
    const int b = NBUF == 2 ? (i & 1) : 0;
    double2* buf = b ? buf1 : buf0;
    mbar_wait(&bar[b], (uint32_t)(NBUF == 2 ? ((i >> 1) & 1) : (i & 1)));
    CS cs{buf + (size_t)(geo.delta - 1) * NFFT};
    dst_pre_inplace<LOGN, NFFT, NT>(a, cs);
    __syncthreads();
    fft_rec<LOGN, NFFT, NT, false, 0, LOGN, TW3>(cs, a.tw);
    dst_post<LOGN, NFFT, NT, false>(cs, scr);
    if (a.vec_out) {
      dst_store<LOGN, NFFT, NT, false>(a, cs, tile_addr<false, C, true>(a, launder(tile)));
    } else {
      dst_store_lines<LOGN, NFFT, NT>(a, cs, tile_addr<false, C, true>(a, launder(tile)));
    }
    // the buffer is refilled by the async proxy: order this thread's generic
    // accesses before it, then make sure every thread is done with it
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (threadIdx.x == 0) {
      const int64_t next = tile + NBUF * (int64_t)gridDim.x;
      if (next < a.ntiles) tma_issue_tile<NFFT>(a, &map, geo, next, buf, &bar[b]);
    }
  }
}

}  // namespace fl
