// Host side of the DST-I transforms: per-length tables, kernel dispatch,
// and the dense sine-matrix path for lengths without an FFT plan.
#include <atomic>
#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <vector>

#include "common.cuh"
#include <cudaTypedefs.h>

#include "dst_fft.cuh"
#include "dst_reg.cuh"
#include "dst_reg10.cuh"
#include "kernels.cuh"

namespace fl {

namespace {

struct Tables {
  double2* tw = nullptr;
  double* sn = nullptr;
  int* perm = nullptr;
  double* sine = nullptr;  // dense n x n unnormalised sine matrix (non-FFT lengths)
};

std::mutex g_mu;
std::map<std::pair<int, int64_t>, Tables> g_tables;  // (device, n)

int ilog2_exact(int64_t v) {
  if (v <= 0 || (v & (v - 1))) return -1;
  int l = 0;
  while ((int64_t(1) << l) < v) ++l;
  return l;
}

bool fft_len_ok(int64_t n) {
  const int lg = ilog2_exact(n + 1);
  return lg >= 2 && lg <= 13;
}

// digit-reversed cell position of every frequency for the DIF plan used on
// the device (radix-8 stages, then one radix-2 or radix-4 stage)
std::vector<int> build_perm(int logn) {
  const int N = 1 << logn;
  std::vector<int> radices;
  for (int s = 0; s < logn / 3; ++s) radices.push_back(8);
  if (logn % 3) radices.push_back(1 << (logn % 3));
  std::vector<int> perm(N);
  for (int k = 0; k < N; ++k) {
    int rem = k, pos = 0, span = N;
    for (int r : radices) {
      const int q = rem % r;
      rem /= r;
      span /= r;
      pos += q * span;
    }
    perm[k] = pos;
  }
  return perm;
}

int make_tables(int64_t n, Tables& t) {
  const long double PI = 3.141592653589793238462643383279502884L;
  if (fft_len_ok(n)) {
    const int logn = ilog2_exact(n + 1);
    const int N = 1 << logn;
    std::vector<double2> tw(N);
    for (int m = 0; m < N; ++m) {
      const long double ang = -2.0L * PI * (long double)m / (long double)N;
      tw[m] = make_double2((double)cosl(ang), (double)sinl(ang));
    }
    std::vector<double> sn(N / 2 + 1);
    for (int j = 0; j <= N / 2; ++j) sn[j] = (double)sinl(PI * (long double)j / (long double)N);
    std::vector<int> perm = build_perm(logn);
    FL_CUDA_TRY(cudaMalloc(&t.tw, sizeof(double2) * N));
    FL_CUDA_TRY(cudaMalloc(&t.sn, sizeof(double) * sn.size()));
    FL_CUDA_TRY(cudaMalloc(&t.perm, sizeof(int) * N));
    FL_CUDA_TRY(cudaMemcpy(t.tw, tw.data(), sizeof(double2) * N, cudaMemcpyHostToDevice));
    FL_CUDA_TRY(cudaMemcpy(t.sn, sn.data(), sizeof(double) * sn.size(), cudaMemcpyHostToDevice));
    FL_CUDA_TRY(cudaMemcpy(t.perm, perm.data(), sizeof(int) * N, cudaMemcpyHostToDevice));
  } else {
    std::vector<double> S((size_t)n * n);
    const long double N1 = (long double)(n + 1);
    for (int64_t k = 0; k < n; ++k)
      for (int64_t j = 0; j < n; ++j) {
        // reduce (j+1)(k+1) mod 2(n+1) exactly before the sine for accuracy
        const int64_t m = ((j + 1) * (k + 1)) % (2 * (n + 1));
        S[(size_t)k * n + j] = (double)sinl(PI * (long double)m / N1);
      }
    FL_CUDA_TRY(cudaMalloc(&t.sine, sizeof(double) * S.size()));
    FL_CUDA_TRY(cudaMemcpy(t.sine, S.data(), sizeof(double) * S.size(), cudaMemcpyHostToDevice));
  }
  return FL_OK;
}

}  // namespace

int get_tables(int64_t n, const Tables** out);

int prepare(int64_t n) {
  const Tables* t;
  return get_tables(n, &t);
}

int get_tables(int64_t n, const Tables** out) {
  FL_ARG_CHECK(n >= 1, "n must be a positive integer, got %lld", (long long)n);
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(g_mu);
  auto key = std::make_pair(dev, n);
  auto it = g_tables.find(key);
  if (it == g_tables.end()) {
    Tables t;
    int rc = make_tables(n, t);
    if (rc != FL_OK) {
      // a failed build frees whatever it had allocated (no leak on retry)
      cudaFree(t.tw);
      cudaFree(t.sn);
      cudaFree(t.perm);
      cudaFree(t.sine);
      return rc;
    }
    it = g_tables.emplace(key, t).first;
  }
  *out = &it->second;
  return FL_OK;
}

namespace {

template <typename K>
int grid_for(K kernel, int nt, size_t smem, int64_t ntiles, int* grid) {
  static std::mutex mu;
  // keyed by (device, kernel): function attributes are set per device
  static std::map<std::pair<int, const void*>, int> occ;
  int blocks = 0;
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  {
    std::lock_guard<std::mutex> lk(mu);
    const auto key = std::make_pair(dev, (const void*)kernel);
    auto it = occ.find(key);
    if (it == occ.end()) {
      if (smem > 48 * 1024)
        FL_CUDA_TRY(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      FL_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, kernel, nt, smem));
      if (blocks < 1) blocks = 1;
      occ[key] = blocks;
    } else {
      blocks = it->second;
    }
  }
  const int64_t cap = (int64_t)blocks * sm_count();
  *grid = (int)(ntiles < cap ? ntiles : cap);
  if (*grid < 1) *grid = 1;
  return FL_OK;
}

template <int LOGN, bool CONTIG, int LOADER, bool MID>
int launch_fft(DstArgs a, cudaStream_t st) {
  using S = DstShape<LOGN>;
  constexpr int NF = MID ? S::NFFT_MID : (LOADER == LOAD_KR ? S::NFFT : S::NFFT_PLAIN);
  constexpr int C = 2 * NF;
  if (CONTIG) {
    a.ntiles = (a.outer + C - 1) / C;
    a.nchunks = 1;
  } else {
    a.nchunks = (a.wv + C - 1) / C;
    a.ntiles = a.outer * a.groups * a.nchunks;
  }
  if (a.ntiles == 0) return FL_OK;
  FL_ARG_CHECK(a.ntiles < (int64_t(1) << 31), "too many DST tiles (%lld)", (long long)a.ntiles);
  if (!CONTIG) {
    a.div_blk = make_fastdiv((uint32_t)(a.groups * a.nchunks));
    a.div_chunk = make_fastdiv((uint32_t)a.nchunks);
  }
  constexpr int NT = MID ? S::NT_MID : (LOADER == LOAD_KR ? S::NT : S::NT_PLAIN);
  constexpr int MINB = MID ? S::MINB_MID : (LOADER == LOAD_KR ? S::MINB : S::MINB_PLAIN);
  constexpr size_t SMEM = MID ? S::smem_mid(NT) : S::smem_n(NT, NF);
  auto kern = k_dst_fft<LOGN, NF, NT, MINB, CONTIG, LOADER, MID>;
  int grid = 0;
  int rc = grid_for(kern, NT, SMEM, a.ntiles, &grid);
  if (rc) return rc;
  kern<<<grid, NT, SMEM, st>>>(a);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

// ---- register-resident N = 512 pass (dst_reg.cuh) -------------------------
bool reg_enabled() {
  static int v = -1;
  if (v < 0) {
    const char* e = getenv("FL_REG");
    v = (e && e[0] == '0') ? 0 : 1;
  }
  return v == 1;
}

PFN_cuTensorMapEncodeTiled_v12000 tma_encoder();

#ifndef FL_REG_TMA
#define FL_REG_TMA 1
#endif

// tensor map of a 16-byte aligned strided input (element (o, g, c, j) at
// o*os + g*gp + c + j*js) with 16-column x 256-row boxes, 128-byte swizzle
bool reg_tensor_map(const DstArgs& a, CUtensorMap* map) {
  auto enc = tma_encoder();
  if (!enc) return false;
  const uint64_t es = sizeof(double);
  const uint64_t rows_b = (uint64_t)a.in_js * es;
  const uint64_t grp_b = a.groups > 1 ? (uint64_t)a.in_gp * es : rows_b * (uint64_t)a.n;
  const uint64_t out_b = a.outer > 1 ? (uint64_t)a.in_os * es : grp_b * (uint64_t)a.groups;
  if (rows_b % 16 || grp_b % 16 || out_b % 16) return false;
  cuuint64_t dims[4] = {(cuuint64_t)a.wv, (cuuint64_t)a.n, (cuuint64_t)a.groups, (cuuint64_t)a.outer};
  cuuint64_t strides[3] = {rows_b, grp_b, out_b};
  cuuint32_t box[4] = {16, 256, 1, 1};
  cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 4, const_cast<double*>(a.x), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// the three output maps of the TMA-store phase (dst_reg.cuh, OutMaps)
bool reg_out_maps(const DstArgs& a, rg::OutMaps* m, int nq = 16) {
  auto enc = tma_encoder();
  if (!enc) return false;
  const uint64_t es = sizeof(double);
  const uint64_t row_b = (uint64_t)a.out_js * es;
  const uint64_t grp_b = a.groups > 1 ? (uint64_t)a.out_gp * es : row_b * 1024;
  const uint64_t out_b = a.outer > 1 ? (uint64_t)a.out_os * es : grp_b * (uint64_t)a.groups;
  if (row_b % 16 || grp_b % 16 || out_b % 16) return false;
  // rows g = 32 qq + ii, qq < nq (= N / 32); halves qq < nq/2 and the rest,
  // the last qq with 31 rows (row N - 1 does not exist)
  cuuint64_t dims[5] = {(cuuint64_t)a.wv, (cuuint64_t)nq, 32, (cuuint64_t)a.groups, (cuuint64_t)a.outer};
  cuuint64_t strides[4] = {32 * row_b, row_b, grp_b, out_b};
  cuuint32_t estr[5] = {1, 1, 1, 1, 1};
  const cuuint32_t hq = (cuuint32_t)(nq / 2);
  const cuuint32_t boxes[3][5] = {{16, hq, 32, 1, 1}, {16, hq - 1, 32, 1, 1}, {16, 1, 31, 1, 1}};
  CUtensorMap* maps[3] = {&m->a, &m->b, &m->c};
  for (int k = 0; k < 3; ++k)
    if (enc(maps[k], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 5, a.y, dims, strides, const_cast<cuuint32_t*>(boxes[k]), estr,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  return true;
}

template <int SIN, int SOUT, bool MID, bool TMA, bool TST>
int launch_reg_k(const DstArgs& a, const CUtensorMap& map, const rg::OutMaps& om, cudaStream_t st) {
  auto kern = rg::k_dst_grp<SIN, SOUT, MID, TMA, TST>;
  constexpr size_t SMEM = rg::grp_smem_bytes();
  // function attributes are per device: one flag bit per device ordinal
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load() & bit)) {
    FL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr_set.fetch_or(bit);
  }
  const int64_t cap = 2 * (int64_t)sm_count();
  const int grid = (int)(a.ntiles < cap ? a.ntiles : cap);
  kern<<<grid, 32 * rg::NWARP, SMEM, st>>>(a, map, om);
  FL_LAUNCH_CHECK();
  return FL_OK;
}

#ifndef FL_REG_TST
#define FL_REG_TST 1
#endif

template <int SIN, int SOUT, bool MID, bool TMA>
int launch_reg_o(const DstArgs& a, const CUtensorMap& map, cudaStream_t st) {
  rg::OutMaps om{};
  if constexpr (SOUT == rg::SIDE_VEC) {
    static int use = -1;
    if (use < 0) {
      const char* e = getenv("FL_REG_TST");
      use = e ? (e[0] != '0') : FL_REG_TST;
    }
    if (use && a.n == 511 && reg_out_maps(a, &om)) return launch_reg_k<SIN, SOUT, MID, TMA, true>(a, map, om, st);
  }
  return launch_reg_k<SIN, SOUT, MID, TMA, false>(a, map, om, st);
}

template <int SIN, int SOUT, bool MID>
int launch_reg(DstArgs a, cudaStream_t st) {
  if (SIN == rg::SIDE_CONTIG) {
    a.ntiles = (a.outer + 15) / 16;
    a.nchunks = 1;
  } else {
    a.nchunks = (a.wv + 15) / 16;
    a.ntiles = a.outer * a.groups * a.nchunks;
  }
  if (a.ntiles == 0) return FL_OK;
  FL_ARG_CHECK(a.ntiles < (int64_t(1) << 31), "too many DST tiles (%lld)", (long long)a.ntiles);
  if (SIN != rg::SIDE_CONTIG) {
    a.div_blk = make_fastdiv((uint32_t)(a.groups * a.nchunks));
    a.div_chunk = make_fastdiv((uint32_t)a.nchunks);
  }
  CUtensorMap map{};
  if constexpr (SIN == rg::SIDE_VEC) {
    static int use = -1;
    if (use < 0) {
      const char* e = getenv("FL_REG_TMA");
      use = e ? (e[0] != '0') : FL_REG_TMA;
    }
    if (use && reg_tensor_map(a, &map)) return launch_reg_o<SIN, SOUT, MID, true>(a, map, st);
  }
  return launch_reg_o<SIN, SOUT, MID, false>(a, map, st);
}

// ---- register-resident N = 1024 passes (dst_reg10.cuh) ---------------------
// strided: 16-byte aligned both sides (TMA loads and stores); contiguous:
// aligned x.  Returns 1 when launched, 0 when the pass is not eligible.
template <int SIN>
int launch_reg10(DstArgs a, cudaStream_t st) {
  if (SIN == rg::SIDE_CONTIG) {
    a.ntiles = (a.outer + 15) / 16;
    a.nchunks = 1;
  } else {
    a.nchunks = (a.wv + 15) / 16;
    a.ntiles = a.outer * a.groups * a.nchunks;
  }
  if (a.ntiles == 0) return 1;
  if (a.ntiles >= (int64_t(1) << 31)) return 0;
  CUtensorMap map{};
  rg::OutMaps om{};
  if (SIN != rg::SIDE_CONTIG) {
    a.div_blk = make_fastdiv((uint32_t)(a.groups * a.nchunks));
    a.div_chunk = make_fastdiv((uint32_t)a.nchunks);
    if (!reg_tensor_map(a, &map) || !reg_out_maps(a, &om, 32)) return 0;
  }
  constexpr int NW = SIN == rg::SIDE_CONTIG ? rg10::CONTIG_NW : 8;
  constexpr int PIECES = 8 / NW;
  if (a.ntiles * PIECES >= (int64_t(1) << 31)) return 0;
  auto kern = rg10::k_dst_reg10<SIN, NW>;
  constexpr size_t SMEM = rg10::smem_bytes<NW>();
  static std::atomic<uint64_t> attr_set{0};
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  const uint64_t bit = uint64_t(1) << (dev & 63);
  if (!(attr_set.load() & bit)) {
    FL_CUDA_TRY(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)SMEM));
    attr_set.fetch_or(bit);
  }
  const int64_t cap = (int64_t)sm_count() * PIECES, pieces = a.ntiles * PIECES;
  const int grid = (int)(pieces < cap ? pieces : cap);
  kern<<<grid, 32 * NW, SMEM, st>>>(a, map, om);
  FL_LAUNCH_CHECK();
  return 1;
}

// ---- tensor-map encoder (driver entry point) -------------------------------
PFN_cuTensorMapEncodeTiled_v12000 tma_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static bool tried = false;
  if (!tried) {
    tried = true;
    cudaDriverEntryPointQueryResult q;
    void* p = nullptr;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

template <bool CONTIG, int LOADER, bool MID>
int dispatch_fft(int logn, const DstArgs& a, cudaStream_t st) {
  switch (logn) {
    case 2: return launch_fft<2, CONTIG, LOADER, MID>(a, st);
    case 3: return launch_fft<3, CONTIG, LOADER, MID>(a, st);
    case 4: return launch_fft<4, CONTIG, LOADER, MID>(a, st);
    case 5: return launch_fft<5, CONTIG, LOADER, MID>(a, st);
    case 6: return launch_fft<6, CONTIG, LOADER, MID>(a, st);
    case 7: return launch_fft<7, CONTIG, LOADER, MID>(a, st);
    case 8: return launch_fft<8, CONTIG, LOADER, MID>(a, st);
    case 9: return launch_fft<9, CONTIG, LOADER, MID>(a, st);
    case 10: return launch_fft<10, CONTIG, LOADER, MID>(a, st);
    case 11: return launch_fft<11, CONTIG, LOADER, MID>(a, st);
    case 12: return launch_fft<12, CONTIG, LOADER, MID>(a, st);
    case 13: return launch_fft<13, CONTIG, LOADER, MID>(a, st);
  }
  set_error("no FFT plan for log2(N) = %d", logn);
  return FL_EINVAL;
}

}  // namespace

// One DST-I pass with explicit input/output layouts (see DstArgs).  FFT
// lengths only; the standard [outer][n][inner] pass is dst_mode below.
int dst_pass(const double* x, double* y, const double* core, int64_t n, bool contig, int64_t outer, int64_t groups,
             int64_t wv, const PassLayout& in, const PassLayout& out, double scale, cudaStream_t st, bool pad_write) {
  FL_ARG_CHECK(n >= 1 && outer >= 0 && groups >= 1 && wv >= 0, "bad DST pass shape");
  FL_ARG_CHECK(fft_len_ok(n), "pass layouts need an FFT length (n+1 a power of two in [4, 8192]), got %lld",
               (long long)n);
  FL_ARG_CHECK(contig || (in.js >= wv && out.js >= wv), "strided pass: row stride below the group width");
  FL_ARG_CHECK(!contig || (in.lp >= n && out.lp >= n && in.lp < (1ll << 31) && out.lp < (1ll << 31)),
               "contiguous pass: line pitch must be in [n, 2^31)");
  if (outer == 0 || wv == 0) return FL_OK;
  const Tables* t = nullptr;
  int rc = get_tables(n, &t);
  if (rc) return rc;
  const int logn = ilog2_exact(n + 1);
  const double nrm = std::sqrt(2.0 / (double)(n + 1));
  DstArgs a{};
  a.x = x;
  a.y = y;
  a.outer = outer;
  a.n = n;
  a.groups = groups;
  a.wv = wv;
  a.in_os = in.os;
  a.in_js = in.js;
  a.in_gp = in.gp;
  a.in_lp = in.lp;
  a.out_os = out.os;
  a.out_js = out.js;
  a.out_gp = out.gp;
  a.out_lp = out.lp;
  a.core = core;
  a.tw = t->tw;
  a.sn = t->sn;
  a.pad_zero = (pad_write && contig && out.lp > n) ? 1 : 0;
  if (!contig) {
    // 16-byte line pairs: aligned base and strides; an odd group width is
    // fine when the layout has room for one more column after the last
    // (a padded row), which the pair access then touches: reads ignore it,
    // writes (only into internal work buffers, pad_write) store the finite
    // transform of the zero-filled partner line
    auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    auto room = [&](const PassLayout& l) { return wv % 2 == 0 || (groups > 1 ? l.gp > wv : l.js > wv); };
    a.vec_in = al(x) && (core == nullptr || al(core)) && in.os % 2 == 0 && in.gp % 2 == 0 && in.js % 2 == 0 &&
               room(in);
    a.vec_out = al(y) && out.os % 2 == 0 && out.gp % 2 == 0 && out.js % 2 == 0 && (wv % 2 == 0 || (pad_write && room(out)));
  }
  if (logn == 10 && reg_enabled() && core == nullptr) {
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    int r = 0;
    a.scale = scale * nrm;
    if (contig && in.lp >= 1023 && in.lp < (1ll << 31) && al16(x)) {
      r = launch_reg10<rg::SIDE_CONTIG>(a, st);
    } else if (!contig && a.vec_in && a.vec_out) {
      r = launch_reg10<rg::SIDE_VEC>(a, st);
    }
    if (r < 0) return -r;
    if (r > 0) return FL_OK;
  }
  if (logn == 9 && reg_enabled()) {
    auto al16 = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
    if (core == nullptr && contig && in.lp >= 511 && al16(x)) {
      a.scale = scale * nrm;
      return launch_reg<rg::SIDE_CONTIG, rg::SIDE_CONTIG, false>(a, st);  // zeroes the padding itself
    }
    if (core == nullptr && !contig) {
      a.scale = scale * nrm;
      if (a.vec_in && a.vec_out) return launch_reg<rg::SIDE_VEC, rg::SIDE_VEC, false>(a, st);
      if (a.vec_in) return launch_reg<rg::SIDE_VEC, rg::SIDE_SCALAR, false>(a, st);
      if (a.vec_out) return launch_reg<rg::SIDE_SCALAR, rg::SIDE_VEC, false>(a, st);
      return launch_reg<rg::SIDE_SCALAR, rg::SIDE_SCALAR, false>(a, st);
    }
  }
  if (contig && a.pad_zero) {
    // CTA kernel: clear the padding after the pass (same stream)
    int rc2 = dst_pass(x, y, core, n, contig, outer, groups, wv, in, out, scale, st, false);
    if (rc2) return rc2;
    FL_CUDA_TRY(cudaMemset2DAsync(y + n, (size_t)out.lp * sizeof(double), 0, (size_t)(out.lp - n) * sizeof(double),
                                  (size_t)outer, st));
    return FL_OK;
  }
  if (core == nullptr) {
    a.scale = scale * nrm;
    if (contig) return dispatch_fft<true, LOAD_PLAIN, false>(logn, a, st);
    // scalar line accesses on either side: lighter twiddle loads (measured)
    return (a.vec_in && a.vec_out) ? dispatch_fft<false, LOAD_PLAIN, false>(logn, a, st)
                                   : dispatch_fft<false, LOAD_PLAIN_TW3, false>(logn, a, st);
  }
  FL_ARG_CHECK(contig, "the fused core pass runs on contiguous lines");
  a.scale = scale * nrm * nrm;
  return dispatch_fft<true, LOAD_PLAIN, true>(logn, a, st);
}

bool fft_length(int64_t n) { return fft_len_ok(n); }

int dst_pass_lanes_mode0(const double* x, double* y, const double* core_l, int64_t groups, double scale,
                         cudaStream_t st) {
  FL_ARG_CHECK(x != nullptr && y != nullptr && core_l != nullptr, "null pointer");
  FL_ARG_CHECK(groups >= 1, "lane-core mode-0 pass: groups must be >= 1");
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  FL_ARG_CHECK(al(x) && al(y) && al(core_l), "lane-core pass: 16-byte aligned buffers required");
  const Tables* t = nullptr;
  int rc = get_tables(511, &t);
  if (rc) return rc;
  const double nrm = std::sqrt(2.0 / 512.0);
  DstArgs a{};
  a.x = x;
  a.y = y;
  a.outer = 1;
  a.n = 511;
  a.groups = groups;
  a.wv = 512;
  a.in_os = a.out_os = 0;
  a.in_js = a.out_js = groups * 512;
  a.in_gp = a.out_gp = 512;
  a.vec_in = a.vec_out = 1;
  a.core = core_l;
  a.tw = t->tw;
  a.sn = t->sn;
  a.scale = scale * nrm * nrm;
  return launch_reg<rg::SIDE_VEC, rg::SIDE_VEC, true>(a, st);
}

int dst_pass_lanes(const double* x, double* y, const double* core_l, int64_t lines, int64_t pitch, double scale,
                   cudaStream_t st) {
  FL_ARG_CHECK(x != nullptr && y != nullptr && core_l != nullptr, "null pointer");
  FL_ARG_CHECK(lines >= 0 && pitch >= 512 && pitch % 2 == 0 && pitch < (1ll << 31),
               "lane-core pass: pitch must be even and >= 512, got %lld", (long long)pitch);
  auto al = [](const void* p) { return ((uintptr_t)p & 15) == 0; };
  FL_ARG_CHECK(al(x) && al(y) && al(core_l), "lane-core pass: 16-byte aligned buffers required");
  if (lines == 0) return FL_OK;
  const Tables* t = nullptr;
  int rc = get_tables(511, &t);
  if (rc) return rc;
  const double nrm = std::sqrt(2.0 / 512.0);
  DstArgs a{};
  a.x = x;
  a.y = y;
  a.outer = lines;
  a.n = 511;
  a.groups = 1;
  a.wv = 1;
  a.in_lp = a.out_lp = pitch;
  a.core = core_l;
  a.tw = t->tw;
  a.sn = t->sn;
  a.scale = scale * nrm * nrm;
  return launch_reg<rg::SIDE_CONTIG, rg::SIDE_CONTIG, true>(a, st);
}

// y = scale * F_n x along the middle axis (optionally core-scaled sandwich)
int dst_mode(const double* x, double* y, int64_t outer, int64_t n, int64_t inner, double scale,
             const double* core, cudaStream_t st) {
  FL_ARG_CHECK(outer >= 0 && n >= 1 && inner >= 1, "bad transform shape (%lld, %lld, %lld)",
               (long long)outer, (long long)n, (long long)inner);
  if (outer == 0) return FL_OK;
  const Tables* t = nullptr;
  int rc = get_tables(n, &t);
  if (rc) return rc;
  if (fft_len_ok(n)) {
    if (inner == 1) {
      const PassLayout l{0, 1, 0, n};
      return dst_pass(x, y, core, n, true, outer, 1, 1, l, l, scale, st);
    }
    const PassLayout l{n * inner, inner, 0, 0};
    if (core == nullptr) return dst_pass(x, y, nullptr, n, false, outer, 1, inner, l, l, scale, st);
    // strided fused pass is not instantiated: transform, scale, transform
    if ((rc = dst_pass(x, y, nullptr, n, false, outer, 1, inner, l, l, 1.0, st))) return rc;
    if ((rc = ew_mul(y, core, y, outer * n * inner, 1.0, st))) return rc;
    return dst_pass(y, y, nullptr, n, false, outer, 1, inner, l, l, scale, st);
  }
  // dense sine-matrix path (DMMA GEMM): y_o = c S x_o, or with a core
  // y_o = c S (core_o .* (nrm S x_o)) with the core folded into the first
  // GEMM's epilogue; x == y goes through a temporary
  const double nrm = std::sqrt(2.0 / (double)(n + 1));
  const int64_t total = outer * n * inner;
  DevBuf tmp;
  if (inner == 1) {
    // lines: Y (outer x n) = X S (S symmetric, read N-major)
    const double* src = x;
    if (x == y || core != nullptr) {
      if ((rc = tmp.alloc(total, st))) return rc;
    }
    if (core != nullptr) {
      if ((rc = gemm_f64_ep(outer, n, n, nrm, x, n, 1, 0, t->sine, n, 1, 0, 0.0, tmp.p, n, 1, 0, 1, core, st)))
        return rc;
      return gemm_f64(outer, n, n, scale * nrm, tmp.p, n, 1, 0, t->sine, n, 1, 0, 0.0, y, n, 1, 0, 1, st);
    }
    if (x == y) {
      FL_CUDA_TRY(cudaMemcpyAsync(tmp.p, x, sizeof(double) * total, cudaMemcpyDeviceToDevice, st));
      src = tmp.p;
    }
    return gemm_f64(outer, n, n, scale * nrm, src, n, 1, 0, t->sine, n, 1, 0, 0.0, y, n, 1, 0, 1, st);
  }
  if (core == nullptr) {
    const double* src = x;
    if (x == y) {
      if ((rc = tmp.alloc(total, st))) return rc;
      FL_CUDA_TRY(cudaMemcpyAsync(tmp.p, x, sizeof(double) * total, cudaMemcpyDeviceToDevice, st));
      src = tmp.p;
    }
    return gemm_f64(n, inner, n, scale * nrm, t->sine, n, 1, 0, src, inner, 1, n * inner, 0.0, y, inner, 1,
                    n * inner, outer, st);
  }
  if ((rc = tmp.alloc(total, st))) return rc;
  if ((rc = gemm_f64_ep(n, inner, n, nrm, t->sine, n, 1, 0, x, inner, 1, n * inner, 0.0, tmp.p, inner, 1,
                        n * inner, outer, core, st)))
    return rc;
  return gemm_f64(n, inner, n, scale * nrm, t->sine, n, 1, 0, tmp.p, inner, 1, n * inner, 0.0, y, inner, 1,
                  n * inner, outer, st);
}

// canonical apply, one mode: out[:, k*S + s] = scale * F(U[:, k] .* Xs[:, s]), out is (n, R*S)
int dst_kr(const double* U, const double* Xs, double* out, int64_t n, int64_t R, int64_t S, double scale,
           cudaStream_t st) {
  FL_ARG_CHECK(n >= 1 && R >= 0 && S >= 0, "bad canonical apply shape");
  if (R == 0 || S == 0) return FL_OK;
  const Tables* t = nullptr;
  int rc = get_tables(n, &t);
  if (rc) return rc;
  if (fft_len_ok(n)) {
    const int logn = ilog2_exact(n + 1);
    DstArgs a{};
    a.y = out;
    a.outer = 1;
    a.n = n;
    a.groups = 1;
    a.wv = R * S;
    a.in_os = a.out_os = n * R * S;
    a.in_js = a.out_js = R * S;
    a.vec_out = ((uintptr_t)out & 15) == 0 && (R * S) % 2 == 0;
    a.U = U;
    a.Xs = Xs;
    a.R = R;
    a.S = S;
    a.tw = t->tw;
    a.sn = t->sn;
    a.scale = scale * std::sqrt(2.0 / (double)(n + 1));
    return dispatch_fft<false, LOAD_KR, false>(logn, a, st);
  }
  rc = kr_expand(U, Xs, out, n, R, S, st);
  if (rc) return rc;
  return dst_mode(out, out, 1, n, R * S, scale, nullptr, st);
}

}  // namespace fl
