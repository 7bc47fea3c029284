// extern "C" entry points of libfraclap_b200.so (see include/fraclap_b200.h).
#include <cstdarg>
#include <cstdio>
#include <mutex>
#include <map>
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace fl {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

// Stream-ordered temporaries come from the device's default memory pool,
// whose release threshold is 0 by default: every synchronisation hands the
// freed blocks back to the driver and the next cudaMallocAsync pays for a
// fresh mapping (~0.3 ms measured per small-SVD call).  Keep up to 1 GiB
// cached in the pool instead (once per device).
int keep_pool_cached() {
  static std::mutex mu;
  static std::map<int, bool> done;
  int dev = 0;
  FL_CUDA_TRY(cudaGetDevice(&dev));
  std::lock_guard<std::mutex> lk(mu);
  if (done[dev]) return FL_OK;
  cudaMemPool_t pool;
  FL_CUDA_TRY(cudaDeviceGetDefaultMemPool(&pool, dev));
  uint64_t cur = 0, want = uint64_t(1) << 30;
  FL_CUDA_TRY(cudaMemPoolGetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &cur));
  if (cur < want) FL_CUDA_TRY(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &want));
  done[dev] = true;
  return FL_OK;
}

int sm_count() {
  static std::mutex mu;
  static std::map<int, int> cache;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return 148;
  std::lock_guard<std::mutex> lk(mu);
  auto it = cache.find(dev);
  if (it != cache.end()) return it->second;
  int v = 0;
  if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) v = 148;
  cache[dev] = v;
  return v;
}

static int check_dims(int d, const int64_t* dims) {
  FL_ARG_CHECK(d == 2 || d == 3, "only tensors of order 2 or 3 are supported, got %d", d);
  for (int l = 0; l < d; ++l) FL_ARG_CHECK(dims[l] >= 1, "mode %d has size %lld", l, (long long)dims[l]);
  return FL_OK;
}

}  // namespace fl

using namespace fl;

extern "C" {

int fl_version(void) { return 1; }

const char* fl_last_error(void) { return g_err; }

int fl_sm_count(void) { return sm_count(); }

int fl_prepare(int64_t n) { return prepare(n); }

int fl_dst1(const double* x, double* y, int64_t outer, int64_t n, int64_t inner, double scale, void* stream) {
  return dst_mode(x, y, outer, n, inner, scale, nullptr, as_stream(stream));
}

int fl_dst1_core(const double* x, double* y, const double* core, int64_t outer, int64_t n, int64_t inner,
                 double scale, void* stream) {
  FL_ARG_CHECK(core != nullptr, "core tensor required");
  return dst_mode(x, y, outer, n, inner, scale, core, as_stream(stream));
}

int fl_basis_apply(const double* Q, int transpose, const double* x, double* y, int64_t outer, int64_t n,
                   int64_t inner, void* stream) {
  FL_ARG_CHECK(n >= 1 && inner >= 1 && outer >= 0, "bad transform shape");
  FL_ARG_CHECK(x != y, "fl_basis_apply does not run in place");
  // forward (transpose=1): y = Q^T x ; inverse: y = Q x
  const int64_t sAm = transpose ? 1 : n, sAk = transpose ? n : 1;
  return gemm_f64(n, inner, n, 1.0, Q, sAm, sAk, 0, x, inner, 1, n * inner, 0.0, y, inner, 1, n * inner, outer,
                  as_stream(stream));
}

int fl_core_eval(double* out, int d, const int64_t* dims, const double* const* mu, int tag, double a, double cm,
                 double cp, int reciprocal, void* stream) {
  int rc = check_dims(d, dims);
  if (rc) return rc;
  return core_eval(out, d, dims, mu, tag, a, cm, cp, reciprocal, as_stream(stream));
}

int fl_cp_to_dense(double* out, int d, const int64_t* dims, int64_t rank, const double* weights,
                   const double* const* factors, void* stream) {
  int rc = check_dims(d, dims);
  if (rc) return rc;
  FL_ARG_CHECK(rank >= 0, "rank must be nonnegative");
  return cp_to_dense(out, d, dims, rank, weights, factors, as_stream(stream));
}

int fl_sinc_factor(double* U, const double* mu, int64_t n, const double* t, int64_t R, double rho_min,
                   void* stream) {
  FL_ARG_CHECK(n >= 1 && R >= 0, "bad sinc factor shape");
  FL_ARG_CHECK(rho_min > 0.0, "rho_min must be positive");
  return sinc_factor(U, mu, n, t, R, rho_min, as_stream(stream));
}

// y = alpha * F diag(core) F x, F = per-mode orthonormal DST-I.
int fl_apply_full(const double* x, double* y, const double* core, int d, const int64_t* dims, double alpha,
                  void* stream) {
  int rc = check_dims(d, dims);
  if (rc) return rc;
  FL_ARG_CHECK(core != nullptr, "core tensor required");
  cudaStream_t st = as_stream(stream);
  if (d == 2) {
    const int64_t n0 = dims[0], n1 = dims[1];
    if ((rc = dst_mode(x, y, 1, n0, n1, 1.0, nullptr, st))) return rc;
    if ((rc = dst_mode(y, y, n0, n1, 1, 1.0, core, st))) return rc;
    return dst_mode(y, y, 1, n0, n1, alpha, nullptr, st);
  }
  const int64_t n0 = dims[0], n1 = dims[1], n2 = dims[2];
  if ((rc = dst_mode(x, y, 1, n0, n1 * n2, 1.0, nullptr, st))) return rc;
  if ((rc = dst_mode(y, y, n0, n1, n2, 1.0, nullptr, st))) return rc;
  if ((rc = dst_mode(y, y, n0 * n1, n2, 1, 1.0, core, st))) return rc;
  if ((rc = dst_mode(y, y, n0, n1, n2, 1.0, nullptr, st))) return rc;
  return dst_mode(y, y, 1, n0, n1 * n2, alpha, nullptr, st);
}

int fl_apply_full_padded(const double* x, double* y, const double* core_p, double* work, int d,
                         const int64_t* dims, int64_t pitch, double alpha, void* stream) {
  int rc = check_dims(d, dims);
  if (rc) return rc;
  FL_ARG_CHECK(core_p != nullptr && work != nullptr, "padded core and work buffer required");
  for (int l = 0; l < d; ++l)
    FL_ARG_CHECK(fft_length(dims[l]), "padded apply needs FFT lengths, mode %d has n = %lld", l, (long long)dims[l]);
  const int64_t nl = dims[d - 1], P = pitch;
  FL_ARG_CHECK(P >= nl, "pitch %lld below the last mode size %lld", (long long)P, (long long)nl);
  cudaStream_t st = as_stream(stream);
  const PassLayout line{0, 1, 0, P};
  if (d == 2) {
    const int64_t n0 = dims[0];
    const PassLayout dense{0, nl, 0, 0}, padded{0, P, 0, 0};
    if ((rc = dst_pass(x, work, nullptr, n0, false, 1, 1, nl, dense, padded, 1.0, st, true))) return rc;
    if ((rc = dst_pass(work, work, core_p, nl, true, n0, 1, 1, line, line, 1.0, st))) return rc;
    return dst_pass(work, y, nullptr, n0, false, 1, 1, nl, padded, dense, alpha, st);
  }
  const int64_t n0 = dims[0], n1 = dims[1];
  const PassLayout dense0{0, n1 * nl, nl, 0}, padded0{0, n1 * P, P, 0};
  const PassLayout mid{n1 * P, P, 0, 0};
  if ((rc = dst_pass(x, work, nullptr, n0, false, 1, n1, nl, dense0, padded0, 1.0, st, true))) return rc;
  if ((rc = dst_pass(work, work, nullptr, n1, false, n0, 1, P, mid, mid, 1.0, st))) return rc;
  if ((rc = dst_pass(work, work, core_p, nl, true, n0 * n1, 1, 1, line, line, 1.0, st))) return rc;
  if ((rc = dst_pass(work, work, nullptr, n1, false, n0, 1, P, mid, mid, 1.0, st))) return rc;
  return dst_pass(work, y, nullptr, n0, false, 1, n1, nl, padded0, dense0, alpha, st);
}

int fl_apply_full_lanes(const double* x, double* y, const double* core_l, double* work, int d, const int64_t* dims,
                        double alpha, void* stream) {
  int rc = check_dims(d, dims);
  if (rc) return rc;
  FL_ARG_CHECK(core_l != nullptr && work != nullptr, "lane-ordered core and work buffer required");
  FL_ARG_CHECK(dims[0] == 511 && dims[d - 1] == 511, "lane-ordered apply needs n_0 = n_last = 511");
  for (int l = 0; l < d; ++l)
    FL_ARG_CHECK(fft_length(dims[l]), "lane apply needs FFT lengths, mode %d has n = %lld", l, (long long)dims[l]);
  const int64_t n0 = 511, nl = 511, P = 512;
  const int64_t n1 = d == 3 ? dims[1] : 1;
  const int64_t lines = n0 * n1;  // lines of the last mode
  cudaStream_t st = as_stream(stream);
  // last mode first, contiguous: dense rows (pitch 511) -> padded rows (512)
  const PassLayout dense_l{0, 1, 0, nl}, pad_l{0, 1, 0, P};
  // (writes the padding position too: pass 2 and the fused pass pair the last
  // column with it in one packed FFT)
  if ((rc = dst_pass(x, work, nullptr, nl, true, lines, 1, 1, dense_l, pad_l, 1.0, st, true))) return rc;
  const PassLayout mid{n1 * P, P, 0, 0};
  if (d == 3 && (rc = dst_pass(work, work, nullptr, n1, false, n0, 1, P, mid, mid, 1.0, st))) return rc;
  // mode 0: forward, core, inverse in one pass
  if ((rc = dst_pass_lanes_mode0(work, work, core_l, n1, 1.0, st))) return rc;
  if (d == 3 && (rc = dst_pass(work, work, nullptr, n1, false, n0, 1, P, mid, mid, 1.0, st))) return rc;
  return dst_pass(work, y, nullptr, nl, true, lines, 1, 1, pad_l, dense_l, alpha, st);
}

int fl_dst1_core_lanes_mode0(const double* x, double* y, const double* core_l, int64_t groups, double scale,
                             void* stream) {
  return dst_pass_lanes_mode0(x, y, core_l, groups, scale, as_stream(stream));
}

int fl_dst1_core_lanes(const double* x, double* y, const double* core_l, int64_t lines, int64_t pitch, double scale,
                       void* stream) {
  return dst_pass_lanes(x, y, core_l, lines, pitch, scale, as_stream(stream));
}

int fl_dst1_pass(const double* x, double* y, const double* core, int64_t n, int contig, int64_t outer,
                 int64_t groups, int64_t width, const int64_t* in_layout, const int64_t* out_layout, double scale,
                 void* stream) {
  FL_ARG_CHECK(in_layout != nullptr && out_layout != nullptr, "layouts required");
  const PassLayout in{in_layout[0], in_layout[1], in_layout[2], in_layout[3]};
  const PassLayout out{out_layout[0], out_layout[1], out_layout[2], out_layout[3]};
  return dst_pass(x, y, core, n, (contig & FL_PASS_CONTIG) != 0, outer, groups, width, in, out, scale,
                  as_stream(stream), (contig & FL_PASS_PAD_WRITE) != 0);
}

int fl_transform_full(const double* x, double* y, int d, const int64_t* dims, double alpha, void* stream) {
  int rc = check_dims(d, dims);
  if (rc) return rc;
  cudaStream_t st = as_stream(stream);
  if (d == 2) {
    const int64_t n0 = dims[0], n1 = dims[1];
    if ((rc = dst_mode(x, y, n0, n1, 1, 1.0, nullptr, st))) return rc;
    return dst_mode(y, y, 1, n0, n1, alpha, nullptr, st);
  }
  const int64_t n0 = dims[0], n1 = dims[1], n2 = dims[2];
  if ((rc = dst_mode(x, y, n0 * n1, n2, 1, 1.0, nullptr, st))) return rc;
  if ((rc = dst_mode(y, y, n0, n1, n2, 1.0, nullptr, st))) return rc;
  return dst_mode(y, y, 1, n0, n1 * n2, alpha, nullptr, st);
}

int fl_svd_batched(const double* A, int batch, int m, int n, double* U, double* S, double* Vt, void* stream) {
  return svd_batched(A, batch, m, n, U, S, Vt, as_stream(stream));
}

int fl_svd_left_pivoted(const double* A, int batch, int k, double* U, double* S, void* stream) {
  return svd_left_pivoted(A, batch, k, U, S, as_stream(stream));
}

int fl_kr_contract(const double* Pa, int64_t a, const double* Pb, int64_t b, int64_t R, const double* Y,
                   int64_t sYr, int64_t sYj, int64_t N, double* out, void* stream) {
  return kr_contract(Pa, a, Pb, b, R, Y, sYr, sYj, N, out, as_stream(stream));
}

int fl_qr_r(int batch, const double* const* M, const int* k, const int64_t* m, const int64_t* rs, const int64_t* cs,
            double* const* R, void* stream) {
  FL_ARG_CHECK(batch == 0 || (M && k && m && rs && cs && R), "fl_qr_r: null argument array");
  return tsqr_r(batch, M, k, m, rs, cs, R, as_stream(stream));
}

int fl_left_sv_wide(int batch, const double* const* M, const int* k, const int64_t* m, const int64_t* rs,
                    const int64_t* cs, double* const* U, double* const* S, void* stream) {
  FL_ARG_CHECK(batch == 0 || (M && k && m && rs && cs && S), "fl_left_sv_wide: null argument array");
  return left_sv_wide(batch, M, k, m, rs, cs, U, S, as_stream(stream));
}

int fl_cp_apply_mode(const double* U, const double* Xs, double* out, int64_t n, int64_t R, int64_t S, double scale,
                     void* stream) {
  return dst_kr(U, Xs, out, n, R, S, scale, as_stream(stream));
}

int fl_cp_gram(int d, const int64_t* n, const double* const* A, int64_t Ra, const double* const* B, int64_t Rb,
               double* H, void* stream) {
  FL_ARG_CHECK(d >= 1 && d <= 3, "order must be 1..3");
  FL_ARG_CHECK(Ra >= 0 && Rb >= 0, "ranks must be nonnegative");
  return gram_hadamard(d, n, A, Ra, B, Rb, H, as_stream(stream));
}

int fl_col_norms(const double* U, int64_t n, int64_t R, double* out, void* stream) {
  FL_ARG_CHECK(n >= 1 && R >= 0, "bad matrix shape");
  return col_norms(U, n, R, out, as_stream(stream));
}

int fl_col_scale(const double* U, const double* nrm, int64_t n, int64_t R, double* V, void* stream) {
  FL_ARG_CHECK(n >= 1 && R >= 0, "bad matrix shape");
  return col_scale(U, nrm, n, R, V, as_stream(stream));
}

int fl_pcg_spectral(const double* b_hat, double* x_hat, double* r, double* p, const double* A, const double* P,
                    int64_t N, double tol, int k_max, double* hist, int* status, void* stream) {
  return pcg_spectral(b_hat, x_hat, r, p, A, P, N, tol, k_max, hist, status, as_stream(stream));
}

int fl_pcg_phase(int phase, const double* b_hat, double* x_hat, double* r, double* p, const double* A,
                 const double* P, int64_t N, double alpha, double beta, double* out, double* work, void* stream) {
  FL_ARG_CHECK(N >= 0, "bad PCG size");
  return pcg_phase(phase, b_hat, x_hat, r, p, A, P, N, alpha, beta, out, work, as_stream(stream));
}

}  // extern "C"
