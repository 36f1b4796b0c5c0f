// Compile-time specialised line FFTs (lengths used by the BASELINE grids and
// the reference's test grids).  Same in-place Stockham scheme as
// fft_engine.cuh, but with N, the radix sequence and every index constant
// known to the compiler: no runtime divisions, no predicated radix slots,
// radix-16/6 codelets so 48 = 16x3, 64 = 16x4, 96 = 16x6 take two passes.
// ncu on the runtime engine showed ~300 instructions per element per line
// FFT at n = 48; this path is what the kernels use whenever a size has a
// plan below (fft_kernels.cu dispatch), the runtime engine otherwise.
#pragma once

#include "grid.cuh"

namespace pwb {

// W_16^q = exp(sgn * 2 pi i q / 16) applied to v
__device__ __forceinline__ double2 w16(double2 v, int q, double sgn) {
  const double c1 = 0.92387953251128675613, s1 = 0.38268343236508977173;
  const double h = 0.70710678118654752440;
  double c, s;
  switch (q) {
    case 0: return v;
    case 1: c = c1; s = s1; break;
    case 2: c = h; s = h; break;
    case 3: c = s1; s = c1; break;
    case 4: return cmul_isgn(v, sgn);
    case 6: c = -h; s = h; break;
    case 9: c = -c1; s = -s1; break;
    default: c = 1.0; s = 0.0; break;
  }
  const double ss = sgn * s;
  return make_double2(v.x * c - v.y * ss, v.x * ss + v.y * c);
}

template <>
struct Dft<16> {
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    double2 y[4][4];
#pragma unroll
    for (int n2 = 0; n2 < 4; ++n2) {
      double2 a[4] = {v[n2], v[4 + n2], v[8 + n2], v[12 + n2]};
      Dft<4>::run(a, sgn);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) y[n2][k1] = w16(a[k1], n2 * k1, sgn);
    }
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 b[4] = {y[0][k1], y[1][k1], y[2][k1], y[3][k1]};
      Dft<4>::run(b, sgn);
#pragma unroll
      for (int k2 = 0; k2 < 4; ++k2) v[k1 + 4 * k2] = b[k2];
    }
  }
};

template <>
struct Dft<6> {
  // 6 = 2 (inner, n1) x 3 (outer, n2): x[3 n1 + n2], X[k1 + 2 k2]
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    const double s3 = 0.86602540378443864676;
    double2 y0[3], y1[3];
#pragma unroll
    for (int n2 = 0; n2 < 3; ++n2) {
      y0[n2] = cadd(v[n2], v[3 + n2]);
      y1[n2] = csub(v[n2], v[3 + n2]);
    }
    // twiddles W6^(n2*k1) for k1 = 1: n2=1 -> (1/2, sgn s3), n2=2 -> (-1/2, sgn s3)
    y1[1] = cmul(y1[1], make_double2(0.5, sgn * s3));
    y1[2] = cmul(y1[2], make_double2(-0.5, sgn * s3));
    Dft<3>::run(y0, sgn);
    Dft<3>::run(y1, sgn);
#pragma unroll
    for (int k2 = 0; k2 < 3; ++k2) {
      v[2 * k2] = y0[k2];
      v[1 + 2 * k2] = y1[k2];
    }
  }
};

template <>
struct Dft<12> {
  // 12 = 4 (inner, n1) x 3 (outer, n2): x[3 n1 + n2], X[k1 + 4 k2];
  // X = sum W4^(n1 k1) W12^(n2 k1) W3^(n2 k2) x
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    const double s3 = 0.86602540378443864676;
    double2 y[3][4];
#pragma unroll
    for (int n2 = 0; n2 < 3; ++n2) {
      double2 a[4] = {v[n2], v[3 + n2], v[6 + n2], v[9 + n2]};
      Dft<4>::run(a, sgn);
#pragma unroll
      for (int k1 = 0; k1 < 4; ++k1) y[n2][k1] = a[k1];
    }
    // W12^q for q = n2 k1 in {1, 2, 3} (n2 = 1) and {2, 4, 6} (n2 = 2)
    y[1][1] = cmul(y[1][1], make_double2(s3, sgn * 0.5));
    y[1][2] = cmul(y[1][2], make_double2(0.5, sgn * s3));
    y[1][3] = cmul_isgn(y[1][3], sgn);
    y[2][1] = cmul(y[2][1], make_double2(0.5, sgn * s3));
    y[2][2] = cmul(y[2][2], make_double2(-0.5, sgn * s3));
    y[2][3] = make_double2(-y[2][3].x, -y[2][3].y);
#pragma unroll
    for (int k1 = 0; k1 < 4; ++k1) {
      double2 b[3] = {y[0][k1], y[1][k1], y[2][k1]};
      Dft<3>::run(b, sgn);
#pragma unroll
      for (int k2 = 0; k2 < 3; ++k2) v[k1 + 4 * k2] = b[k2];
    }
  }
};

// One compile-time Stockham pass (radix R, sub-transform size NS) over whole
// lines, one butterfly per thread per round.
// vm (first pass only, optional): input element e of line l is multiplied by
// vs * vm[e * vld + l] as it is loaded (fuses the pointwise V(r) product of
// the H apply into the forward transform).
template <int N, int R, int NS, int NT>
__device__ __forceinline__ void spass(double2* __restrict__ s, int nlines, int es, int ls,
                                      const int* __restrict__ lbase,
                                      const double2* __restrict__ tw, bool inv, bool line_major,
                                      const double* __restrict__ vm = nullptr, int vld = 0,
                                      double vs = 1.0) {
  constexpr int NBF = N / R;
  constexpr int LPR = (NT / NBF) > 0 ? (NT / NBF) : 1;   // whole lines per round
  constexpr int TWS = N / (NS * R);
  const double sgn = inv ? 1.0 : -1.0;
  const int tid = threadIdx.x;
  int l_in, j;
  if (line_major) {
    l_in = tid / NBF;
    j = tid - l_in * NBF;
  } else {
    j = tid / LPR;
    l_in = tid - j * LPR;
  }
  const bool lane_ok = (l_in < LPR) && (j < NBF);
  const int k = j % NS;
  const int o0 = (j - k) * R + k;
  // twiddles for this thread's butterfly are the same in every round
  double2 w[R];
  if (NS > 1 && lane_ok) {
#pragma unroll
    for (int r = 1; r < R; ++r) {
      double2 t = __ldg(&tw[r * k * TWS]);
      if (inv) t.y = -t.y;
      w[r] = t;
    }
  }
  // MR rounds of LPR lines share one load phase and one store phase (one
  // barrier pair): fewer barriers and MR * R independent smem loads in flight
  // for the small radices (radix-3 pass of 48 = 16 x 3 over 64 lines: 2
  // barriers instead of 8).
  constexpr int MR = (12 / R) > 1 ? (12 / R) : 1;
#pragma unroll 1
  for (int l0 = 0; l0 < nlines; l0 += LPR * MR) {
    double2 v[MR][R];
    int base[MR];
    bool ok[MR];
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      const int l = l0 + m * LPR + l_in;
      ok[m] = lane_ok && (l < nlines);
      base[m] = 0;
      if (ok[m]) {
        base[m] = lbase ? lbase[l] : l * ls;
#pragma unroll
        for (int r = 0; r < R; ++r) v[m][r] = s[base[m] + (j + r * NBF) * es];
        if (NS == 1 && vm) {
          // multiplier stored element-major (vm[e * vld + l]): consecutive lines are
          // consecutive threads, so these loads coalesce
          const double* vl = vm + l;
#pragma unroll
          for (int r = 0; r < R; ++r)
            v[m][r] = cscale(v[m][r], vs * vl[(size_t)(j + r * NBF) * vld]);   // smem or global
        }
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MR; ++m) {
      if (ok[m]) {
        if (NS > 1) {
#pragma unroll
          for (int r = 1; r < R; ++r) v[m][r] = cmul(v[m][r], w[r]);
        }
        Dft<R>::run(v[m], sgn);
#pragma unroll
        for (int r = 0; r < R; ++r) s[base[m] + (o0 + r * NS) * es] = v[m][r];
      }
    }
    __syncthreads();
  }
}

template <int N, int NS, int... Rs>
struct Passes;

template <int N, int NS>
struct Passes<N, NS> {
  template <int NT>
  static __device__ __forceinline__ void run(double2*, int, int, int, const int*, const double2*,
                                            bool, bool, const double* = nullptr, int = 0,
                                            double = 1.0) {}
};

template <int N, int NS, int R, int... Rest>
struct Passes<N, NS, R, Rest...> {
  template <int NT>
  static __device__ __forceinline__ void run(double2* s, int nl, int es, int ls, const int* lb,
                                            const double2* tw, bool inv, bool lm,
                                            const double* vm = nullptr, int vld = 0,
                                            double vs = 1.0) {
    spass<N, R, NS, NT>(s, nl, es, ls, lb, tw, inv, lm, vm, vld, vs);
    Passes<N, NS * R, Rest...>::template run<NT>(s, nl, es, ls, lb, tw, inv, lm);
  }
};

// radix plans (first pass first)
template <int N>
struct StaticPlan {
  static constexpr bool ok = false;
};
#define PWB_PLAN(N, ...)                                                                  \
  template <>                                                                            \
  struct StaticPlan<N> {                                                                 \
    static constexpr bool ok = true;                                                     \
    template <int NT>                                                                    \
    static __device__ __forceinline__ void run(double2* s, int nl, int es, int ls,       \
                                              const int* lb, const double2* tw, bool inv, \
                                              int lm = -1, const double* vm = nullptr,  \
                                              int vld = 0, double vs = 1.0) {           \
      Passes<N, 1, __VA_ARGS__>::template run<NT>(s, nl, es, ls, lb, tw, inv,            \
                                                  lm < 0 ? es == 1 : lm == 1, vm, vld, vs); \
    }                                                                                    \
  };
PWB_PLAN(6, 6)
PWB_PLAN(8, 8)
PWB_PLAN(12, 4, 3)
PWB_PLAN(16, 16)
PWB_PLAN(24, 8, 3)
PWB_PLAN(32, 8, 4)
#ifdef PWB_PLAN48_86
PWB_PLAN(48, 8, 6)
#else
PWB_PLAN(48, 16, 3)
#endif
PWB_PLAN(64, 16, 4)
PWB_PLAN(96, 16, 6)
PWB_PLAN(216, 6, 6, 6)
PWB_PLAN(320, 16, 4, 5)
#undef PWB_PLAN

// line-FFT policies used to template the transform kernels
//   run(g, s, nlines, es, ls, lbase, inv, lm, vm, vld, vs)
// lm: line mapping (-1 auto = along the line when es == 1, 0 across lines,
// 1 along); vm/vld/vs: optional pointwise real multiplier applied to the
// input (element e of line l times vs * vm[e * vld + l]).  N = the compile-time
// length (0 for the runtime engine).
template <int NT>
__device__ __forceinline__ void premultiply(double2* s, int n, int nl, int es, int ls,
                                            const double* vm, int vld, double vs) {
  for (int i = threadIdx.x; i < nl * n; i += NT) {
    const int l = i / n, e = i - l * n;
    s[l * ls + e * es] = cscale(s[l * ls + e * es], vs * vm[(size_t)e * vld + l]);
  }
  __syncthreads();
}

struct DynX {
  static constexpr int N = 0;
  template <int NT>
  static __device__ __forceinline__ void run(const GridDev& g, double2* s, int nl, int es,
                                            int ls, const int* lb, bool inv, int = -1,
                                            const double* vm = nullptr, int vld = 0,
                                            double vs = 1.0) {
    if (vm) premultiply<NT>(s, g.px.n, nl, es, ls, vm, vld, vs);
    fft_lines<NT>(s, g.px, nl, es, ls, lb, inv);
  }
};
struct DynY {
  static constexpr int N = 0;
  template <int NT>
  static __device__ __forceinline__ void run(const GridDev& g, double2* s, int nl, int es,
                                            int ls, const int* lb, bool inv, int = -1,
                                            const double* = nullptr, int = 0, double = 1.0) {
    fft_lines<NT>(s, g.py, nl, es, ls, lb, inv);
  }
};
struct DynZ {
  static constexpr int N = 0;
  template <int NT>
  static __device__ __forceinline__ void run(const GridDev& g, double2* s, int nl, int es,
                                            int ls, const int* lb, bool inv, int = -1,
                                            const double* = nullptr, int = 0, double = 1.0) {
    fft_lines<NT>(s, g.pz, nl, es, ls, lb, inv);
  }
};
template <int NN>
struct StX {
  static constexpr int N = NN;
  template <int NT>
  static __device__ __forceinline__ void run(const GridDev& g, double2* s, int nl, int es,
                                            int ls, const int* lb, bool inv, int lm = -1,
                                            const double* vm = nullptr, int vld = 0,
                                            double vs = 1.0) {
    StaticPlan<NN>::template run<NT>(s, nl, es, ls, lb, g.px.tw, inv, lm, vm, vld, vs);
  }
};
template <int NN>
struct StY {
  static constexpr int N = NN;
  template <int NT>
  static __device__ __forceinline__ void run(const GridDev& g, double2* s, int nl, int es,
                                            int ls, const int* lb, bool inv, int lm = -1,
                                            const double* = nullptr, int = 0, double = 1.0) {
    StaticPlan<NN>::template run<NT>(s, nl, es, ls, lb, g.py.tw, inv, lm);
  }
};
template <int NN>
struct StZ {
  static constexpr int N = NN;
  template <int NT>
  static __device__ __forceinline__ void run(const GridDev& g, double2* s, int nl, int es,
                                            int ls, const int* lb, bool inv, int lm = -1,
                                            const double* = nullptr, int = 0, double = 1.0) {
    StaticPlan<NN>::template run<NT>(s, nl, es, ls, lb, g.pz.tw, inv, lm);
  }
};

}  // namespace pwb
