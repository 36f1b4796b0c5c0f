// Shared-memory line-FFT engine (complex FP64, mixed radix 2/3/4/5/8).
//
// A CTA transforms a set of lines that live in shared memory, in place, by
// Stockham autosort passes.  Each pass reads a group of whole lines into
// registers (K butterflies of radix R per thread), synchronises, and writes
// the twiddled R-point DFT outputs back to their autosorted positions, so a
// single shared buffer suffices (no ping-pong) -- a 96x96 complex plane is
// 147 KB and a 32x320 plane 164 KB, both within one SM's 227 KB.
//
// Conventions: forward = exp(-2 pi i jk/n) (numpy fftn), inverse =
// exp(+2 pi i jk/n), both unnormalised.  tw[m] = exp(-2 pi i m/n).
#pragma once

#include "common.cuh"

namespace pwb {

constexpr int kMaxPasses = 8;

// radices packed 4 bits per pass, first pass in the low bits, 0 terminates
struct LinePlan {
  int n;
  unsigned code;
  const double2* tw;  // device table, n entries
};

// ---------------------------------------------------------------------------
// In-register R-point DFTs.  sgn = +1 for inverse, -1 for forward.
template <int R>
struct Dft;

template <>
struct Dft<2> {
  static __device__ __forceinline__ void run(double2* v, double) {
    double2 a = v[0], b = v[1];
    v[0] = cadd(a, b);
    v[1] = csub(a, b);
  }
};

template <>
struct Dft<4> {
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    double2 s02 = cadd(v[0], v[2]), d02 = csub(v[0], v[2]);
    double2 s13 = cadd(v[1], v[3]), d13 = cmul_isgn(csub(v[1], v[3]), sgn);
    v[0] = cadd(s02, s13);
    v[2] = csub(s02, s13);
    v[1] = cadd(d02, d13);
    v[3] = csub(d02, d13);
  }
};

template <>
struct Dft<8> {
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    const double h = 0.70710678118654752440;
    double2 e[4] = {v[0], v[2], v[4], v[6]};
    double2 o[4] = {v[1], v[3], v[5], v[7]};
    Dft<4>::run(e, sgn);
    Dft<4>::run(o, sgn);
    // twiddles w8^q, w8 = exp(sgn * 2 pi i / 8)
    double2 o1 = make_double2(h * (o[1].x - sgn * o[1].y), h * (o[1].y + sgn * o[1].x));
    double2 o2 = cmul_isgn(o[2], sgn);
    double2 o3 = make_double2(h * (-o[3].x - sgn * o[3].y), h * (-o[3].y + sgn * o[3].x));
    v[0] = cadd(e[0], o[0]);
    v[4] = csub(e[0], o[0]);
    v[1] = cadd(e[1], o1);
    v[5] = csub(e[1], o1);
    v[2] = cadd(e[2], o2);
    v[6] = csub(e[2], o2);
    v[3] = cadd(e[3], o3);
    v[7] = csub(e[3], o3);
  }
};

template <>
struct Dft<3> {
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    const double s3 = 0.86602540378443864676;
    double2 t = cadd(v[1], v[2]);
    double2 m = make_double2(v[0].x - 0.5 * t.x, v[0].y - 0.5 * t.y);
    double2 u = cmul_isgn(csub(v[1], v[2]), sgn * s3);
    v[0] = cadd(v[0], t);
    v[1] = cadd(m, u);
    v[2] = csub(m, u);
  }
};

template <>
struct Dft<5> {
  static __device__ __forceinline__ void run(double2* v, double sgn) {
    const double c1 = 0.30901699437494742410;   // cos(2pi/5)
    const double c2 = -0.80901699437494742410;  // cos(4pi/5)
    const double s1 = 0.95105651629515357212;   // sin(2pi/5)
    const double s2 = 0.58778525229247312917;   // sin(4pi/5)
    double2 t1 = cadd(v[1], v[4]), d1 = csub(v[1], v[4]);
    double2 t2 = cadd(v[2], v[3]), d2 = csub(v[2], v[3]);
    double2 a0 = v[0];
    double2 b1 = make_double2(a0.x + c1 * t1.x + c2 * t2.x, a0.y + c1 * t1.y + c2 * t2.y);
    double2 b2 = make_double2(a0.x + c2 * t1.x + c1 * t2.x, a0.y + c2 * t1.y + c1 * t2.y);
    double2 q1 = make_double2(s1 * d1.x + s2 * d2.x, s1 * d1.y + s2 * d2.y);
    double2 q2 = make_double2(s2 * d1.x - s1 * d2.x, s2 * d1.y - s1 * d2.y);
    q1 = cmul_isgn(q1, sgn);
    q2 = cmul_isgn(q2, sgn);
    v[0] = make_double2(a0.x + t1.x + t2.x, a0.y + t1.y + t2.y);
    v[1] = cadd(b1, q1);
    v[4] = csub(b1, q1);
    v[2] = cadd(b2, q2);
    v[3] = csub(b2, q2);
  }
};

// ---------------------------------------------------------------------------
// One Stockham pass of radix R (runtime, one of 2,3,4,5,8) over `nlines`
// lines of length n in smem.
//   element e of line l lives at s[base(l) + e * es],
//   base(l) = lbase ? lbase[l] : l * ls.
// line_major: consecutive threads walk along a line (use when es == 1);
// otherwise consecutive threads walk across lines (use when lines are
// adjacent in memory).  Whole lines are processed per register round (K
// butterflies per thread), which makes the in-place update race-free.  The
// register tile is always K x 8 complex with predicated slots so that all
// radices share one allocation (mixing radix-templated passes in one kernel
// made ptxas allocate them additively and spill).
template <int K, int NT>
__device__ __forceinline__ void fft_pass(double2* __restrict__ s, int R, int n, int ns,
                                         int nlines, int es, int ls,
                                         const int* __restrict__ lbase,
                                         const double2* __restrict__ tw, bool inv,
                                         bool line_major) {
  const int nbf = n / R;
  int lpr = (NT * K) / nbf;
  if (lpr < 1) lpr = 1;
  const int tw_step = n / (ns * R);
  const double sgn = inv ? 1.0 : -1.0;
#pragma unroll 1
  for (int l0 = 0; l0 < nlines; l0 += lpr) {
    const int lr = min(lpr, nlines - l0);
    const int total = lr * nbf;
    double2 v[K][8];
    int wb[K], jj[K];
#pragma unroll
    for (int q = 0; q < K; ++q) {
      const int b = q * NT + (int)threadIdx.x;
      wb[q] = -1;
      jj[q] = 0;
      if (b < total) {
        int l, j;
        if (line_major) {
          l = b / nbf;
          j = b - l * nbf;
        } else {
          j = b / lr;
          l = b - j * lr;
        }
        l += l0;
        const int base = lbase ? lbase[l] : l * ls;
        wb[q] = base;
        jj[q] = j;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < R) v[q][r] = s[base + (j + r * nbf) * es];
      }
    }
    __syncthreads();
#pragma unroll
    for (int q = 0; q < K; ++q) {
      if (wb[q] >= 0) {
        const int j = jj[q];
        const int k = j % ns;
        if (ns > 1) {
#pragma unroll
          for (int r = 1; r < 8; ++r) {
            if (r < R) {
              double2 w = __ldg(&tw[r * k * tw_step]);
              if (inv) w.y = -w.y;
              v[q][r] = cmul(v[q][r], w);
            }
          }
        }
        switch (R) {
          case 8: Dft<8>::run(v[q], sgn); break;
          case 4: Dft<4>::run(v[q], sgn); break;
          case 2: Dft<2>::run(v[q], sgn); break;
          case 3: Dft<3>::run(v[q], sgn); break;
          default: Dft<5>::run(v[q], sgn); break;
        }
        const int o0 = (j - k) * R + k;
#pragma unroll
        for (int r = 0; r < 8; ++r)
          if (r < R) s[wb[q] + (o0 + r * ns) * es] = v[q][r];
      }
    }
    __syncthreads();
  }
}

// Full in-place FFT of a set of lines (all passes).  Must be called by all
// threads of the CTA (contains __syncthreads).
template <int NT>
__device__ __forceinline__ void fft_lines(double2* s, const LinePlan& pl, int nlines, int es,
                                          int ls, const int* lbase, bool inv) {
  const bool line_major = (es == 1);
  const int n = pl.n;
  const double2* tw = pl.tw;
  unsigned code = pl.code;
  int ns = 1;
#pragma unroll 1
  while (code) {
    const int R = code & 15u;
    code >>= 4;
    fft_pass<2, NT>(s, R, n, ns, nlines, es, ls, lbase, tw, inv, line_major);
    ns *= R;
  }
}

}  // namespace pwb
