// Kernel-variant dispatch: compile-time FFT codelets (fft_static.cuh) for the
// cube shapes in use, the runtime engine (fft_engine.cuh) for any other shape.
#pragma once

#include "fft_static.cuh"
#include "grid.cuh"

namespace pwb {

// Two-pass plans N = R1 x R2 for the fused pencil / accumulation kernels
// (k_pencil_h, k_drho_h): pass R1 with NS = 1, then R2 with NS = R1.
template <int N>
struct TwoPass {
  static constexpr bool ok = false;
};
template <>
struct TwoPass<48> {   // 8 x 6: register-resident radix-16 lines spill (measured 1.63 vs 1.46 us/band)
  static constexpr bool ok = true;
  static constexpr int R1 = 8, R2 = 6;
};
template <>
struct TwoPass<64> {
  static constexpr bool ok = true;
  static constexpr int R1 = 16, R2 = 4;
};
template <>
struct TwoPass<96> {   // 8 x 12: radix-16 lines held in registers spilled at 80 registers
  static constexpr bool ok = true;  // (ncu at 96^3: STL/LDL a quarter of the pencil's stalls)
#ifdef PWB_TWOPASS96_16x6
  static constexpr int R1 = 16, R2 = 6;
#else
  static constexpr int R1 = 8, R2 = 12;
#endif
};

// ----------------------------------------------------------------------------
// dispatch: compile-time codelets for the cube shapes in use, runtime engine otherwise
#define PWB_PLANE_SHAPES(X) X(6, 6) X(8, 8) X(12, 12) X(16, 16) X(24, 24) X(32, 32) \
  X(48, 48) X(64, 64) X(96, 96) X(32, 320)
#define PWB_PENCIL_SIZES(X) X(6) X(8) X(12) X(16) X(24) X(32) X(48) X(64) X(96) X(216)

template <class F>
inline void plane_variant(const pwb_grid* g, F&& f) {
  const int ny = g->ny, nz = g->nz;
#define PWB_PV(Y, Z)                          \
  if (ny == Y && nz == Z) {                   \
    f(StY<Y>(), StZ<Z>());                    \
    return;                                   \
  }
  PWB_PLANE_SHAPES(PWB_PV)
#undef PWB_PV
  f(DynY(), DynZ());
}

template <class F>
inline void pencil_variant(const pwb_grid* g, F&& f) {
  const int nx = g->nx;
#define PWB_XV(X)     \
  if (nx == X) {      \
    f(StX<X>());      \
    return;           \
  }
  PWB_PENCIL_SIZES(PWB_XV)
#undef PWB_XV
  f(DynX());
}

}  // namespace pwb
