// Shared helpers for the fraclap B200 kernels (sm_100a, fp64 throughout).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/fraclap_b200.h"

namespace fl {

// thread-local last error string, surfaced through fl_last_error()
void set_error(const char* fmt, ...);

#define FL_CUDA_TRY(expr)                                                     \
  do {                                                                        \
    cudaError_t _e = (expr);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::fl::set_error("%s:%d: %s: %s", __FILE__, __LINE__, #expr,             \
                      cudaGetErrorString(_e));                                \
      (void)cudaGetLastError(); /* reset the thread's (non-sticky) error */   \
      return _e == cudaErrorMemoryAllocation ? FL_ENOMEM : FL_ECUDA;          \
    }                                                                         \
  } while (0)

#define FL_ARG_CHECK(cond, ...)                                               \
  do {                                                                        \
    if (!(cond)) {                                                            \
      ::fl::set_error(__VA_ARGS__);                                           \
      return FL_EINVAL;                                                       \
    }                                                                         \
  } while (0)

#define FL_LAUNCH_CHECK()                                                     \
  do {                                                                        \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      ::fl::set_error("%s:%d: kernel launch: %s", __FILE__, __LINE__,         \
                      cudaGetErrorString(_e));                                \
      return FL_ECUDA;                                                        \
    }                                                                         \
  } while (0)

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

// raise the default memory pool's release threshold (once per device)
int keep_pool_cached();

// stream-ordered device temporary, freed on every exit path
struct DevBuf {
  double* p = nullptr;
  cudaStream_t st = nullptr;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  int alloc(int64_t count, cudaStream_t s) {
    st = s;
    if (int rc = keep_pool_cached()) return rc;
    FL_CUDA_TRY(cudaMallocAsync(&p, sizeof(double) * (size_t)count, s));
    return FL_OK;
  }
  ~DevBuf() {
    if (p) cudaFreeAsync(p, st);
  }
};

int sm_count();

__device__ __forceinline__ double2 cadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__device__ __forceinline__ double2 csub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(fma(a.x, b.x, -a.y * b.y), fma(a.x, b.y, a.y * b.x));
}
// multiply by -i
__device__ __forceinline__ double2 cmul_mi(double2 a) { return make_double2(a.y, -a.x); }

}  // namespace fl
