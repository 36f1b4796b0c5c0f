// Common helpers for libpwb200 (sm_100a): complex FP64 arithmetic, status
// codes, error propagation across the C-ABI, launch accounting.
#pragma once

#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <utility>

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

// Global -> smem staging with U loads in flight per thread.  A plain
// `sm[f(i)] = src[g(i)]` loop serialises on every load's latency (the store
// may alias the generic source pointer, so loads cannot be hoisted); ncu showed
// long-scoreboard stalls dominating the pencil and plane passes.
template <int U, int NTH, class Load, class Store>
__device__ __forceinline__ void staged_copy(int n, Load load, Store store) {
  for (int i0 = threadIdx.x; i0 < n; i0 += U * NTH) {
    double2 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * NTH;
      if (i < n) v[u] = load(i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int i = i0 + u * NTH;
      if (i < n) store(i, v[u]);
    }
  }
}

// --- programmatic dependent launch (PDL) ---------------------------------------
// Kernels of the CG iteration are launched with programmatic stream
// serialisation: the next kernel's launch and prologue overlap the tail of the
// previous one.  Every kernel launched this way calls pdl_wait() before it
// touches global memory written or read by its predecessor (so before any
// global access at all), which also keeps the completion chain transitive.
// (An explicit early griddepcontrol.launch_dependents was measured 2% slower at
// configs[1]: the successor's parked blocks take SM slots from the running grid.)
__device__ __forceinline__ void pdl_wait() {
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
extern bool g_pdl;   // false when PWB_NO_PDL is set (A/B measurement)

template <typename... KArgs, typename... Args>
inline cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                            cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = g_pdl ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Cooperative launch (all CTAs guaranteed co-resident, or the launch fails with
// cudaErrorCooperativeLaunchTooLarge) for kernels with a software grid barrier.
template <typename... KArgs, typename... Args>
inline cudaError_t launch_coop(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                               cudaStream_t st, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

}  // namespace pwb
