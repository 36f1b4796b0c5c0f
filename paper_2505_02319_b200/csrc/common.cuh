// Common helpers for libpwb200 (sm_100a): complex FP64 arithmetic, status
// codes, error propagation across the C-ABI, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <string>

#include "../../include/pwb200.h"

namespace pwb {

// --- thread-local error message + status -----------------------------------
void set_error(const std::string& msg);
const char* last_error();

// count of kernels launched by this library (bench.py reports it as
// gpu_launches); incremented at every launch site.
extern unsigned long long g_launches;
inline void count_launch(int n = 1) { g_launches += (unsigned long long)n; }

#define PWB_CUDA(call)                                                        \
  do {                                                                        \
    cudaError_t _e = (call);                                                  \
    if (_e != cudaSuccess) {                                                  \
      ::pwb::set_error(std::string(#call) + ": " + cudaGetErrorString(_e));   \
      return PWB_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

#define PWB_LAUNCH_CHECK()                                                    \
  do {                                                                        \
    ::pwb::count_launch();                                                    \
    cudaError_t _e = cudaGetLastError();                                      \
    if (_e != cudaSuccess) {                                                  \
      ::pwb::set_error(std::string("kernel launch: ") + cudaGetErrorString(_e)); \
      return PWB_ERR_CUDA;                                                    \
    }                                                                         \
  } while (0)

#define PWB_TRY(call)                                                         \
  do {                                                                        \
    int _s = (call);                                                          \
    if (_s != PWB_OK) return _s;                                              \
  } while (0)

inline int fail(int code, const std::string& msg) {
  set_error(msg);
  return code;
}

// --- complex helpers ----------------------------------------------------------
__host__ __device__ __forceinline__ double2 cadd(double2 a, double2 b) {
  return make_double2(a.x + b.x, a.y + b.y);
}
__host__ __device__ __forceinline__ double2 csub(double2 a, double2 b) {
  return make_double2(a.x - b.x, a.y - b.y);
}
__host__ __device__ __forceinline__ double2 cmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ double2 cscale(double2 a, double s) {
  return make_double2(a.x * s, a.y * s);
}
// a * (i * sgn)
__host__ __device__ __forceinline__ double2 cmul_isgn(double2 a, double sgn) {
  return make_double2(-sgn * a.y, sgn * a.x);
}
__host__ __device__ __forceinline__ double2 cconj(double2 a) { return make_double2(a.x, -a.y); }

constexpr int kSM = 148;   // B200 SM count (grid sizing)

}  // namespace pwb
