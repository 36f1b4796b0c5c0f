// Batched, pruned 3-D FFT kernels for sphere <-> cube transforms (sm_100a).
//
// A sphere -> real-space transform of one band is split into
//   plane pass  (one CTA per active x plane): scatter the sphere points of
//               that plane into a shared-memory y-z plane, z-FFTs on the
//               active y lines only, y-FFTs on every z line, write the plane;
//   pencil pass (one CTA per tile of y-z points): x-FFT of length nx whose
//               input is zero outside the active planes.
// The H apply fuses inverse-x, *V(r)/n_g and forward-x in ONE pencil pass,
// and the forward plane pass fuses the sphere gather with the kinetic and
// eigenvalue-shift epilogue, so H psi costs three passes over the pruned
// plane buffer ("Kernels").  Only nxa of nx planes (the sphere
// occupies |ix| <= ~N/4 of the 2x-oversampled cube) are ever stored.
#include "dispatch.cuh"
#include "tma.cuh"

namespace pwb {

constexpr int NT = 256;
#ifndef PWB_FFT_MINB
#define PWB_FFT_MINB 3   // min resident CTAs per SM for the H-apply kernels (80-register cap; measured best)
#endif

// ----------------------------------------------------------------------------
// Threads per plane CTA: planes too large for 3 resident CTAs per SM (96 x 96,
// 32 x 320: 150-170 KB of smem, one CTA per SM) get 512 threads so that an SM
// still has 16 warps to hide the global and barrier latency (ncu at 96^3:
// 12% warps active, 1.7 TB/s with 256 threads).
#ifndef PWB_PLANE_BIG_NT
#define PWB_PLANE_BIG_NT 512
#endif
template <class FY, class FZ>
constexpr int plane_nt() {
  return (FY::N * FZ::N > 4800) ? PWB_PLANE_BIG_NT : NT;
}

// plane pass, inverse: sphere rows -> W[b][p]
template <class FY, class FZ, int PT = plane_nt<FY, FZ>()>
__global__ void __launch_bounds__(PT, PT == NT ? PWB_FFT_MINB : 1) k_plane_inv(GridDev g, const double2* __restrict__ psi,
                                                  const double2* __restrict__ psi2,
                                                  const int* __restrict__ band_k, double scale,
                                                  double2* __restrict__ W,
                                                  const int* __restrict__ rows,
                                                  const int* __restrict__ nact) {
  pdl_wait();
  extern __shared__ double2 sm[];
  if (nact && (int)blockIdx.y >= *nact) return;   // device-side row count (graph replay)
  const int p = blockIdx.x;
  const int b = blockIdx.y;                     // plane-buffer slot
  const int row = rows ? rows[b] : b;           // sphere row (active-row compaction)
  const int k = band_k ? band_k[row] : 0;
  // plane geometry: compile-time for the codelet sizes (strides fold into addressing)
  const int ny = FY::N ? FY::N : g.ny;
  const int nz = FZ::N ? FZ::N : g.nz;
  const int nyz = ny * nz;
  const int nyp = FY::N ? (FY::N % 2 == 0 ? FY::N + 1 : FY::N) : g.nyp;   // odd smem stride
  const int s0 = g.xr[k * (g.nxa + 1) + p];
  const int s1 = g.xr[k * (g.nxa + 1) + p + 1];
  const double2* src = psi + (size_t)row * g.nbp;
  const int* pp = g.ppp + (size_t)k * g.nbp;
  // The plane's sphere coefficients (a few per thread) are loaded BEFORE the smem plane
  // is zeroed and in one batch: the CTA used to zero, synchronise, and then pay one
  // global-load latency per loop trip (index + value) before its first FFT; without
  // the butterflies the H apply still took 83% of its time.
  constexpr int GB = 4;   // loads in flight per thread; more points loop
  int gi[GB];
  double2 gv[GB];
#pragma unroll
  for (int u = 0; u < GB; ++u) {
    const int s = s0 + threadIdx.x + u * PT;
    if (s < s1) {
      gi[u] = pp[s];
      gv[u] = psi2 ? cadd(src[s], psi2[(size_t)row * g.nbp + s]) : src[s];
    }
  }
  for (int i = threadIdx.x; i < nz * nyp; i += PT) sm[i] = make_double2(0.0, 0.0);
  __syncthreads();
#pragma unroll
  for (int u = 0; u < GB; ++u)
    if (s0 + threadIdx.x + u * PT < s1) sm[gi[u]] = cscale(gv[u], scale);
  for (int s = s0 + threadIdx.x + GB * PT; s < s1; s += PT) {
    const double2 v = psi2 ? cadd(src[s], psi2[(size_t)row * g.nbp + s]) : src[s];
    sm[pp[s]] = cscale(v, scale);
  }
  __syncthreads();
  FZ::template run<PT>(g, sm, g.nya, nyp, 0, g.ya, true);    // z lines of active y
  FY::template run<PT>(g, sm, nz, 1, nyp, nullptr, true, 0);  // y lines, threads across lines
  double2* dst = W + ((size_t)b * g.nxa + p) * nyz;
  for (int i = threadIdx.x; i < nyz; i += PT) {
    const int z = i / ny;
    dst[i] = sm[i + z * (nyp - ny)];
  }
}

// plane pass, forward: W[b][p] -> sphere rows with epilogue
//   out[s] = a * F(W)[pp[s]] + (kin[s] - shift[b]) * psi_in[s]
template <class FY, class FZ, int PT = plane_nt<FY, FZ>()>
__global__ void __launch_bounds__(PT, PT == NT ? PWB_FFT_MINB : 1) k_plane_fwd(GridDev g, const double2* __restrict__ W,
                                                  const int* __restrict__ band_k, double a,
                                                  const double2* __restrict__ psi_in,
                                                  const double* __restrict__ shift,
                                                  double2* __restrict__ out,
                                                  const int* __restrict__ rows,
                                                  const int* __restrict__ nact) {
  pdl_wait();
  extern __shared__ double2 sm[];
  if (nact && (int)blockIdx.y >= *nact) return;
  const int p = blockIdx.x;
  const int slot = blockIdx.y;                  // plane-buffer slot
  const int b = rows ? rows[slot] : slot;       // sphere row
  const int k = band_k ? band_k[b] : 0;
  const int ny = FY::N ? FY::N : g.ny;
  const int nz = FZ::N ? FZ::N : g.nz;
  const int nyz = ny * nz;
  const int nyp = FY::N ? (FY::N % 2 == 0 ? FY::N + 1 : FY::N) : g.nyp;
  const double2* srcw = W + ((size_t)slot * g.nxa + p) * nyz;
  staged_copy<8, PT>(
      nyz, [&](int i) { return __ldg(&srcw[i]); },
      [&](int i, double2 v) { sm[i + (i / ny) * (nyp - ny)] = v; });
  __syncthreads();
  FY::template run<PT>(g, sm, nz, 1, nyp, nullptr, false, 0);  // y lines, every z
  FZ::template run<PT>(g, sm, g.nya, nyp, 0, g.ya, false);       // z lines of active y
  const int s0 = g.xr[k * (g.nxa + 1) + p];
  const int s1 = g.xr[k * (g.nxa + 1) + p + 1];
  const int* pp = g.ppp + (size_t)k * g.nbp;
  const double* kin = g.kin + (size_t)k * g.nbp;
  double2* dst = out + (size_t)b * g.nbp;
  const double sh = shift ? shift[b] : 0.0;
  if (psi_in) {
    const double2* pin = psi_in + (size_t)b * g.nbp;
    // all of a thread's index / psi / kinetic loads first, then the smem reads and stores
    // (one global-load latency at the end of the CTA instead of one per loop trip)
    constexpr int GB = 4;
    for (int sb = s0 + threadIdx.x; sb < s1; sb += GB * PT) {
      int gi[GB];
      double2 q[GB];
      double d[GB];
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const int s = sb + u * PT;
        if (s < s1) {
          gi[u] = pp[s];
          q[u] = pin[s];
          d[u] = kin[s] - sh;
        }
      }
#pragma unroll
      for (int u = 0; u < GB; ++u) {
        const int s = sb + u * PT;
        if (s < s1) {
          const double2 v = sm[gi[u]];
          dst[s] = make_double2(a * v.x + d[u] * q[u].x, a * v.y + d[u] * q[u].y);
        }
      }
    }
  } else {
    for (int s = s0 + threadIdx.x; s < s1; s += PT) dst[s] = cscale(sm[pp[s]], a);
  }
}

// ----------------------------------------------------------------------------
// pencil pass.  IN: 0 = W rows (plane list xin), 1 = natural complex,
// 2 = natural real.  OUT: 0 = W rows (plane list xout), 1 = natural complex,
// 2 = natural real part (+ LDA term).  mode: 0 none, 1 fwd, 2 inv,
// 3 inv -> *v*vscale -> fwd.
struct PencilArgs {
  const double2* win;
  const double2* cin;
  const double* rin;
  const int* xin;
  int nxin;
  size_t in_stride;  // elements per band
  const double* v;
  double vscale;
  int mode;
  double2* wout;
  double2* cout;
  double* rout;
  const int* xout;
  int nxout;
  size_t out_stride;
  double oscale;
  const double* lda_v;    // optional: rout += lda_c * max(rho,1e-10)^(-2/3) * lda_v
  const double* lda_rho;
  double lda_c;
  const int* nact;        // optional device row count: blocks with b >= *nact exit
};

// TC: compile-time tile (the codelet sizes' default 3072 / N), 0 = runtime g.tile;
// with it every smem stride and index division folds to constants (ncu: integer
// index arithmetic was half the pencil's instructions).
template <int IN, int OUT, class FX, int TC = 0>
__global__ void __launch_bounds__(NT, PWB_FFT_MINB) k_pencil(GridDev g, PencilArgs a) {
  pdl_wait();
  extern __shared__ double2 sm[];
  const int T = TC ? TC : g.tile;
  const int Tp = TC ? (TC % 2 == 0 ? TC + 1 : TC) : g.tilep;
  const int nyz = g.nyz;
  const int nx = FX::N ? FX::N : g.nx;   // compile-time for the codelet sizes
  const int t0 = blockIdx.x * T;
  const int b = blockIdx.y;
  if (a.nact && b >= *a.nact) return;
  const int nt = min(T, nyz - t0);
  if (IN == 0) {
    if (a.nxin < nx) {
      // zero only the x rows outside the (contiguous, wrapped) active range
      const int x0 = a.xin[a.nxin - 1] + 1;
      const int nz_rows = nx - a.nxin;
      for (int i = threadIdx.x; i < nz_rows * Tp; i += NT) {
        const int q = i / Tp, t = i - q * Tp;
        int x = x0 + q;
        if (x >= nx) x -= nx;
        sm[x * Tp + t] = make_double2(0.0, 0.0);
      }
    }
    if (a.mode == 3) {   // stage this tile's V(r) (x-major) with the W loads: off the FFT path
      double* smv = reinterpret_cast<double*>(sm + nx * Tp);
      const double* vsrc = a.v + t0;
      for (int i0 = threadIdx.x; i0 < nx * T; i0 += 8 * NT) {
        double v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          const int i = i0 + u * NT, x = i / T, t = i - x * T;
          v[u] = (i < nx * T && t < nt) ? __ldg(&vsrc[(size_t)x * nyz + t]) : 0.0;
        }
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (i0 + u * NT < nx * T) smv[i0 + u * NT] = v[u];
      }
    }
    const double2* src = a.win + (size_t)b * a.in_stride;
    staged_copy<6, NT>(
        a.nxin * T,
        [&](int i) {
          const int p = i / T, t = i - p * T;
          return t < nt ? __ldg(&src[(size_t)p * nyz + t0 + t]) : make_double2(0.0, 0.0);
        },
        [&](int i, double2 v) {
          const int p = i / T;
          sm[a.xin[p] * Tp + (i - p * T)] = v;
        });
  } else {
    const size_t base = (size_t)b * a.in_stride + (size_t)t0 * nx;
    staged_copy<8, NT>(
        nt * nx,
        [&](int i) {
          return (IN == 1) ? __ldg(&a.cin[base + i]) : make_double2(__ldg(&a.rin[base + i]), 0.0);
        },
        [&](int i, double2 v) {
          const int t = i / nx;
          sm[(i - t * nx) * Tp + t] = v;
        });
  }
  __syncthreads();
  if (a.mode == 1) {
    FX::template run<NT>(g, sm, nt, Tp, 1, nullptr, false);
  } else if (a.mode >= 2) {
    FX::template run<NT>(g, sm, nt, Tp, 1, nullptr, true);
    if (a.mode == 3)   // V(r)/n_g applied inside the first pass of the forward transform
      FX::template run<NT>(g, sm, nt, Tp, 1, nullptr, false, -1,
                           reinterpret_cast<const double*>(sm + nx * Tp), T, a.vscale);
  }
  if (OUT == 0) {
    double2* dst = a.wout + (size_t)b * a.out_stride;
    for (int i = threadIdx.x; i < a.nxout * T; i += NT) {
      const int p = i / T, t = i - p * T;
      if (t < nt) dst[(size_t)p * nyz + t0 + t] = cscale(sm[a.xout[p] * Tp + t], a.oscale);
    }
  } else if (OUT == 3) {   // x-major complex cube [x][yz] (psi(r) cache of the accumulation)
    double2* dst = a.cout + (size_t)b * a.out_stride;
    for (int i = threadIdx.x; i < nx * T; i += NT) {
      const int x = i / T, t = i - x * T;
      if (t < nt) dst[(size_t)x * nyz + t0 + t] = cscale(sm[x * Tp + t], a.oscale);
    }
  } else {
    const size_t base = (size_t)b * a.out_stride + (size_t)t0 * nx;
    for (int i = threadIdx.x; i < nt * nx; i += NT) {
      const int t = i / nx, x = i - t * nx;
      const double2 v = sm[x * Tp + t];
      if (OUT == 1) {
        a.cout[base + i] = cscale(v, a.oscale);
      } else {
        double r = v.x * a.oscale;
        if (a.lda_v) {
          const size_t gi = (size_t)t0 * nx + i;
          const double rho = fmax(a.lda_rho[gi], 1e-10);
          r += a.lda_c * pow(rho, -2.0 / 3.0) * a.lda_v[gi];
        }
        a.rout[base + i] = r;
      }
    }
  }
}

// ----------------------------------------------------------------------------
// full plane pass on all y/z lines of Wf[v][x][z][y].
//   mode 0: transform (forward: y then z; inverse: z then y)
//   mode 1: Hartree  D = 4 pi / |G|^2 (0 at G = 0)     fwd -> *D -> inv
//   mode 2: Kerker   D = |G|^2/(|G|^2+alpha^2) (1 at G=0)
template <class FY, class FZ>
__global__ void __launch_bounds__(NT) k_plane_full(GridDev g, double2* __restrict__ Wf, int mode,
                                                   double param, int inverse) {
  pdl_wait();
  extern __shared__ double2 sm[];
  const int x = blockIdx.x;
  const int v = blockIdx.y;
  const int nyz = g.nyz;
  const int ny = FY::N ? FY::N : g.ny;
  const int nyp = g.nyp;
  double2* pl = Wf + ((size_t)v * g.nx + x) * nyz;
  staged_copy<8, NT>(
      nyz, [&](int i) { return pl[i]; },
      [&](int i, double2 v) { sm[i + (i / ny) * (nyp - ny)] = v; });
  __syncthreads();
  if (mode == 0 && inverse) {
    FZ::template run<NT>(g, sm, g.ny, nyp, 1, nullptr, true);
    FY::template run<NT>(g, sm, g.nz, 1, nyp, nullptr, true, 0);
  } else {
    FY::template run<NT>(g, sm, g.nz, 1, nyp, nullptr, false, 0);
    FZ::template run<NT>(g, sm, g.ny, nyp, 1, nullptr, false);
  }
  if (mode != 0) {
    const double* g2 = g.g2w + (size_t)x * nyz;
    for (int i = threadIdx.x; i < nyz; i += NT) {
      const double q = g2[i];
      double d;
      if (mode == 1) d = (q == 0.0) ? 0.0 : 4.0 * M_PI / q;
      else d = (q == 0.0) ? 1.0 : q / (q + param * param);
      const int j = i + (i / ny) * (nyp - ny);
      sm[j] = cscale(sm[j], d);
    }
    __syncthreads();
    FZ::template run<NT>(g, sm, g.ny, nyp, 1, nullptr, true);
    FY::template run<NT>(g, sm, g.nz, 1, nyp, nullptr, true, 0);
  }
  for (int i = threadIdx.x; i < nyz; i += NT) pl[i] = sm[i + (i / ny) * (nyp - ny)];
}

// ----------------------------------------------------------------------------
// H-apply pencil for two-pass lengths N = R1 x R2 (48 = 16 x 3, 64 = 16 x 4, ...):
// inverse x-FFT, * V(r)/n_g, forward x-FFT with 2 smem round trips instead of 6.
//   A: W rows (active x only, zeros elsewhere) straight from global into the
//      radix-R1 inverse pass (NS = 1) -> smem
//   B: radix-R2 inverse pass (NS = R1, natural-order outputs x = j + r R1),
//      * V, then the forward transform's FIRST pass in the reversed plan
//      R2 x R1 (radix R2, NS = 1), which reads exactly those x: all in registers
//   C: radix-R1 forward pass (NS = R2) -> the active x rows straight to global.
// Three barriers per CTA (the generic path: about twelve).  Same twiddle table
// and DFT codelets as the generic passes; the forward plan order differs, so
// results agree with it to rounding, not bitwise.  (TwoPass plans: dispatch.cuh.)
template <int N>
#ifndef PWB_PENCIL_H_MINB
#define PWB_PENCIL_H_MINB 3   // 80-register cap; 3 CTAs/SM (smem 75 KB each)
#endif
// 96 (8 x 12): 2 CTAs/SM leave 128 registers for the radix-12 pass (no spill;
// 13.7 vs 14.0 us/band at 96^3); 48 / 64 keep 3 CTAs/SM
__global__ void __launch_bounds__(NT, (N == 96 ? 2 : PWB_PENCIL_H_MINB)) k_pencil_h(GridDev g, PencilArgs a) {
  constexpr int R1 = TwoPass<N>::R1, R2 = TwoPass<N>::R2;
  constexpr int TC = 3072 / N, TP = (TC % 2 == 0) ? TC + 1 : TC;
  constexpr int NB1 = N / R1;                 // radix-R1 butterflies per line (= R2)
  constexpr int LP1 = NT / NB1;               // lines per round, passes A and C
  constexpr int LP2 = NT / R1;                // lines per round, pass B
  constexpr int MB = (TC + LP2 - 1) / LP2;    // pass-B rounds held in registers
  static_assert(NB1 == R2, "two-pass plan");
  pdl_wait();
  extern __shared__ double2 sm[];
  double* smv = reinterpret_cast<double*>(sm + N * TP);   // V(r) tile, x-major [x][TC]
  const int nyz = g.nyz;
  const int t0 = blockIdx.x * TC;
  const int b = blockIdx.y;
  if (a.nact && b >= *a.nact) return;
  const int nt = min(TC, nyz - t0);
  const int x0 = a.xin[0], nact_x = a.nxin;   // active x: contiguous wrapped range from x0
  const int tid = threadIdx.x;
  // V tile (consumed in pass B; the loads overlap pass A)
  for (int i0 = tid; i0 < N * TC; i0 += 8 * NT) {
    double v[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int i = i0 + u * NT, x = i / TC, t = i - x * TC;
      v[u] = (i < N * TC && t < nt) ? __ldg(&a.v[(size_t)x * nyz + t0 + t]) : 0.0;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u)
      if (i0 + u * NT < N * TC) smv[i0 + u * NT] = v[u];
  }
  // ---- A: inverse pass 1 (radix R1, NS = 1), inputs from global
  {
    const int j = tid / LP1, li = tid - j * LP1;
    const double2* src = a.win + (size_t)b * a.in_stride;
    if (j < NB1) {
      for (int l = li; l < TC; l += LP1) {
        double2 v[R1];
#pragma unroll
        for (int r = 0; r < R1; ++r) {
          const int x = j + r * NB1;
          int p = x - x0;
          if (p < 0) p += N;
          v[r] = (p < nact_x && l < nt) ? __ldg(&src[(size_t)p * nyz + t0 + l])
                                        : make_double2(0.0, 0.0);
        }
        Dft<R1>::run(v, 1.0);
#pragma unroll
        for (int r = 0; r < R1; ++r) sm[(j * R1 + r) * TP + l] = v[r];
      }
    }
  }
  __syncthreads();
  // ---- B: inverse pass 2 (radix R2, NS = R1) -> * V -> forward pass 1 (radix R2, NS = 1)
  {
    const int j = tid / LP2, li = tid - j * LP2;   // j in [0, R1)
    // twiddles (TWS = N / (NS R) = 1, inverse: conjugate): held across the MB
    // rounds for the small radices, read from L1 per use for radix 12
    constexpr bool kHoldW = R2 <= 8;
    double2 w[kHoldW ? R2 : 1];
    if constexpr (kHoldW) {
#pragma unroll
      for (int r = 1; r < R2; ++r) {
        const double2 t = __ldg(&g.px.tw[r * j]);
        w[r] = make_double2(t.x, -t.y);
      }
    }
    double2 v[MB][R2];
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const int l = m * LP2 + li;
      if (l < TC) {
#pragma unroll
        for (int r = 0; r < R2; ++r) v[m][r] = sm[(j + r * R1) * TP + l];
      }
    }
    __syncthreads();
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const int l = m * LP2 + li;
      if (l < TC) {
#pragma unroll
        for (int r = 1; r < R2; ++r) {
          if constexpr (kHoldW) {
            v[m][r] = cmul(v[m][r], w[r]);
          } else {
            const double2 t = __ldg(&g.px.tw[r * j]);
            v[m][r] = cmul(v[m][r], make_double2(t.x, -t.y));
          }
        }
        Dft<R2>::run(v[m], 1.0);
#pragma unroll
        for (int r = 0; r < R2; ++r) v[m][r] = cscale(v[m][r], a.vscale * smv[(j + r * R1) * TC + l]);
        Dft<R2>::run(v[m], -1.0);
#pragma unroll
        for (int r = 0; r < R2; ++r) sm[(j * R2 + r) * TP + l] = v[m][r];
      }
    }
  }
  __syncthreads();
  // ---- C: forward pass 2 (radix R1, NS = R2), active outputs straight to global
  {
    const int j = tid / LP1, li = tid - j * LP1;   // j in [0, R2)
    if (j < NB1) {
      double2* dst = a.wout + (size_t)b * a.out_stride;
      for (int l = li; l < TC; l += LP1) {
        double2 v[R1];
#pragma unroll
        for (int r = 0; r < R1; ++r) v[r] = sm[(j + r * R2) * TP + l];
#pragma unroll
        for (int r = 1; r < R1; ++r)   // twiddles (TWS = 1, forward) from L1: registers are tight
          v[r] = cmul(v[r], __ldg(&g.px.tw[r * j]));
        Dft<R1>::run(v, -1.0);
        if (l < nt) {
#pragma unroll
          for (int r = 0; r < R1; ++r) {
            int p = j + r * R2 - x0;
            if (p < 0) p += N;
            if (p < nact_x) dst[(size_t)p * nyz + t0 + l] = cscale(v[r], a.oscale);
          }
        }
      }
    }
  }
}

// ----------------------------------------------------------------------------
// Pipelined H-apply pencil: the same three passes as k_pencil_h, but each CTA is
// persistent over a contiguous range of (band, tile) items and a producer warp
// streams the NEXT items' active W rows into a ring of shared-memory stages with
// TMA bulk copies (one copy per active x row, completion on an mbarrier), so the
// HBM reads of item n+1 overlap the FFTs of item n.  ncu on k_pencil_h (48^3):
// the top stall was pass A waiting on its global loads (long scoreboard) at
// ~1.9 TB/s.  V(r) is read from L2 in pass B (x-major, coalesced) to leave the
// shared memory for the stages: 2 CTAs of 9 warps per SM.
constexpr int kHpStages = 2;
#ifndef PWB_PENCIL_VPRE
#define PWB_PENCIL_VPRE 1   // V(r) loads hoisted to the start of pass B
#endif

template <int N>
struct PencilHp {
  static constexpr int TC = 3072 / N, TP = (TC % 2 == 0) ? TC + 1 : TC;
  // double2 elements: work area, then kHpStages stages of nxa x TC
  static size_t smem(int nxa) {
    return ((size_t)N * TP + (size_t)kHpStages * nxa * TC) * 16 + 2 * kHpStages * 8 + 16;
  }
};

template <int N>
__global__ void __launch_bounds__(NT + 32, 2) k_pencil_hp(GridDev g, PencilArgs a, int nb_host,
                                                          int ntiles) {
  constexpr int R1 = TwoPass<N>::R1, R2 = TwoPass<N>::R2;
  constexpr int TC = PencilHp<N>::TC, TP = PencilHp<N>::TP;
  constexpr int NB1 = N / R1;
  constexpr int LP1 = NT / NB1;
  constexpr int LP2 = NT / R1;
  constexpr int MB = (TC + LP2 - 1) / LP2;
  constexpr int NW = NT / 32;
  static_assert(NB1 == R2, "two-pass plan");
  pdl_wait();
  extern __shared__ __align__(128) double2 sm[];
  const int nxa = a.nxin;
  double2* stages = sm + N * TP;
  uint64_t* full = reinterpret_cast<uint64_t*>(stages + (size_t)kHpStages * nxa * TC);
  uint64_t* empty = full + kHpStages;
  const int nyz = g.nyz;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nb = a.nact ? *a.nact : nb_host;
  const int nitems = nb * ntiles;   // item = band * ntiles + tile
  const int per = (nitems + gridDim.x - 1) / gridDim.x;
  const int i0 = blockIdx.x * per, i1 = min(nitems, i0 + per);
  if (tid == 0) {
    for (int s = 0; s < kHpStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (w == NW) {   // producer warp
    for (int item = i0, n = 0; item < i1; ++item, ++n) {
      const int s = n % kHpStages;
      if (n >= kHpStages) mbar_wait(&empty[s], ((n / kHpStages) + 1) & 1);
      const int b = item / ntiles, t0 = (item - b * ntiles) * TC;
      const int nt = min(TC, nyz - t0);
      if (lane == 0) mbar_expect_tx(&full[s], (uint32_t)(nxa * nt * 16));
      __syncwarp();
      const double2* src = a.win + (size_t)b * a.in_stride + t0;
      double2* dst = stages + (size_t)s * nxa * TC;
      for (int p = lane; p < nxa; p += 32)
        bulk_g2s(dst + p * TC, src + (size_t)p * nyz, (uint32_t)(nt * 16), &full[s]);
    }
    return;
  }
  const int x0 = a.xin[0];
  for (int item = i0, n = 0; item < i1; ++item, ++n) {
    const int s = n % kHpStages;
    const int b = item / ntiles, t0 = (item - b * ntiles) * TC;
    const int nt = min(TC, nyz - t0);
    const double2* st = stages + (size_t)s * nxa * TC;
    mbar_wait(&full[s], (n / kHpStages) & 1);
    // ---- A: inverse pass 1 (radix R1, NS = 1) from the stage
    {
      const int j = tid / LP1, li = tid - j * LP1;
      if (j < NB1) {
        for (int l = li; l < TC; l += LP1) {
          double2 v[R1];
#pragma unroll
          for (int r = 0; r < R1; ++r) {
            int p = j + r * NB1 - x0;
            if (p < 0) p += N;
            v[r] = (p < nxa && l < nt) ? st[p * TC + l] : make_double2(0.0, 0.0);
          }
          Dft<R1>::run(v, 1.0);
#pragma unroll
          for (int r = 0; r < R1; ++r) sm[(j * R1 + r) * TP + l] = v[r];
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with stage s
    asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
    // ---- B: inverse pass 2 -> * V (from L2) -> forward pass 1, in registers
    {
      const int j = tid / LP2, li = tid - j * LP2;
      // V(r) loads issued first: their L2 latency overlaps the smem reads and the
      // inverse radix-R2 arithmetic below
      double vv[MB][R2];
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        const int l = m * LP2 + li;
#pragma unroll
        for (int r = 0; r < R2; ++r)
#if PWB_PENCIL_VPRE
          vv[m][r] = (l < TC && l < nt) ? __ldg(&a.v[(size_t)(j + r * R1) * nyz + t0 + l]) : 0.0;
#else
          vv[m][r] = 0.0;
#endif
      }
      double2 v[MB][R2];
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        const int l = m * LP2 + li;
        if (l < TC) {
#pragma unroll
          for (int r = 0; r < R2; ++r) v[m][r] = sm[(j + r * R1) * TP + l];
        }
      }
      asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
#pragma unroll
      for (int m = 0; m < MB; ++m) {
        const int l = m * LP2 + li;
        if (l < TC) {
#pragma unroll
          for (int r = 1; r < R2; ++r) {
            const double2 t = __ldg(&g.px.tw[r * j]);   // inverse: conjugate
            v[m][r] = cmul(v[m][r], make_double2(t.x, -t.y));
          }
          Dft<R2>::run(v[m], 1.0);
#pragma unroll
          for (int r = 0; r < R2; ++r) {
#if !PWB_PENCIL_VPRE
            vv[m][r] = l < nt ? __ldg(&a.v[(size_t)(j + r * R1) * nyz + t0 + l]) : 0.0;
#endif
            v[m][r] = cscale(v[m][r], a.vscale * vv[m][r]);
          }
          Dft<R2>::run(v[m], -1.0);
#pragma unroll
          for (int r = 0; r < R2; ++r) sm[(j * R2 + r) * TP + l] = v[m][r];
        }
      }
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");
    // ---- C: forward pass 2 (radix R1, NS = R2) -> active rows to global
    {
      const int j = tid / LP1, li = tid - j * LP1;
      if (j < NB1) {
        double2* dst = a.wout + (size_t)b * a.out_stride;
        for (int l = li; l < TC; l += LP1) {
          double2 v[R1];
#pragma unroll
          for (int r = 0; r < R1; ++r) v[r] = sm[(j + r * R2) * TP + l];
#pragma unroll
          for (int r = 1; r < R1; ++r) v[r] = cmul(v[r], __ldg(&g.px.tw[r * j]));
          Dft<R1>::run(v, -1.0);
          if (l < nt) {
#pragma unroll
            for (int r = 0; r < R1; ++r) {
              int p = j + r * R2 - x0;
              if (p < 0) p += N;
              if (p < nxa) dst[(size_t)p * nyz + t0 + l] = cscale(v[r], a.oscale);
            }
          }
        }
      }
    }
    asm volatile("bar.sync 1, %0;\n" ::"n"(NT) : "memory");   // work area reused next item
  }
}

size_t plane_smem(const pwb_grid* g) { return (size_t)g->nz * g->dev.nyp * sizeof(double2); }
size_t pencil_smem(const pwb_grid* g) { return (size_t)g->nx * g->dev.tilep * sizeof(double2); }
// W -> W pencil with the V(r) multiply: + the tile's V values (x-major doubles)
static size_t pencil_smem_v(const pwb_grid* g) {
  return pencil_smem(g) + (size_t)g->nx * g->dev.tile * sizeof(double);
}

static int tiles(const pwb_grid* g) { return (g->nyz + g->dev.tile - 1) / g->dev.tile; }

static int check_band_count(int n) {
  if (n < 0 || n > 65535) return fail(PWB_ERR_VALUE, "band batch must be 0..65535 rows");
  return PWB_OK;
}

int launch_plane_inv(pwb_grid* g, int nband, const int* band_k, const double2* psi, double scale,
                     double2* W, const int* rows, const int* nact) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  dim3 grid(g->nxa, nband);
  plane_variant(g, [&](auto fy, auto fz) {
    (void)launch_k(k_plane_inv<decltype(fy), decltype(fz)>, grid,
                   plane_nt<decltype(fy), decltype(fz)>(), plane_smem(g), g->stream, 
        g->dev, psi, nullptr, band_k, scale, W, rows, nact);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_plane_inv2(pwb_grid* g, int nband, const int* band_k, const double2* a,
                      const double2* b, double2* W) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  dim3 grid(g->nxa, nband);
  plane_variant(g, [&](auto fy, auto fz) {
    (void)launch_k(k_plane_inv<decltype(fy), decltype(fz)>, grid,
                   plane_nt<decltype(fy), decltype(fz)>(), plane_smem(g), g->stream, 
        g->dev, a, b, band_k, 1.0, W, nullptr, nullptr);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_plane_fwd(pwb_grid* g, int nband, const int* band_k, const double2* W, double a,
                     const double2* psi_in, const double* shift, double2* out, const int* rows,
                     const int* nact) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  dim3 grid(g->nxa, nband);
  plane_variant(g, [&](auto fy, auto fz) {
    (void)launch_k(k_plane_fwd<decltype(fy), decltype(fz)>, grid,
                   plane_nt<decltype(fy), decltype(fz)>(), plane_smem(g), g->stream, 
        g->dev, W, band_k, a, psi_in, shift, out, rows, nact);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

static PencilArgs empty_args() {
  PencilArgs a;
  memset(&a, 0, sizeof(a));
  a.vscale = 1.0;
  a.oscale = 1.0;
  return a;
}

// vt[x * nyz + t] = v[t * nx + x]: the x-major copy of a real grid vector used
// by the fused V(r) multiply of the pencil pass (coalesced loads)
__global__ void k_transpose_v(int nx, int nyz, const double* __restrict__ v,
                              double* __restrict__ vt) {
  pdl_wait();
  __shared__ double tile[32][33];
  const int t0 = blockIdx.x * 32, x0 = blockIdx.y * 32;
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int t = t0 + i, x = x0 + threadIdx.x;
    if (t < nyz && x < nx) tile[i][threadIdx.x] = v[(size_t)t * nx + x];
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += 8) {
    const int x = x0 + i, t = t0 + threadIdx.x;
    if (t < nyz && x < nx) vt[(size_t)x * nyz + t] = tile[threadIdx.x][i];
  }
}

int launch_transpose_v(pwb_grid* g, const double* v, double* vt) {
  dim3 grid((g->nyz + 31) / 32, (g->nx + 31) / 32);
  (void)launch_k(k_transpose_v, grid, dim3(32, 8), 0, g->stream, g->nx, g->nyz, v, vt);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

// v: x-major (launch_transpose_v) real multiplier
int launch_pencil_vmul(pwb_grid* g, int nband, double2* W, const double* v, double vscale,
                       const int* nact) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  PencilArgs a = empty_args();
  a.nact = nact;
  a.win = W;
  a.xin = g->dev.xa;
  a.nxin = g->nxa;
  a.in_stride = (size_t)g->nxa * g->nyz;
  a.v = v;
  a.vscale = vscale;
  a.mode = 3;
  a.wout = W;
  a.xout = g->dev.xa;
  a.nxout = g->nxa;
  a.out_stride = a.in_stride;
  dim3 grid(tiles(g), nband);
  static const bool generic_only = getenv("PWB_NO_PENCIL_H") != nullptr;   // A/B measurement
  static const bool no_hp = getenv("PWB_NO_PENCIL_HP") != nullptr;          // A/B measurement
  pencil_variant(g, [&](auto fx) {
    using FX = decltype(fx);
    constexpr int TC = FX::N ? 3072 / FX::N : 0;
    if constexpr (TwoPass<FX::N>::ok) {
      if (!generic_only && !no_hp && g->dev.tile == TC) {
        const int nt = tiles(g);
        const int gsz = (int)std::min<long>((long)nt * nband, 2L * kSM);
        (void)launch_k(k_pencil_hp<FX::N>, gsz, NT + 32, PencilHp<FX::N>::smem(g->nxa), g->stream,
                       g->dev, a, nband, nt);
        return;
      }
      if (!generic_only && g->dev.tile == TC) {
        (void)launch_k(k_pencil_h<FX::N>, grid, NT, pencil_smem_v(g), g->stream, g->dev, a);
        return;
      }
    }
    if (TC && g->dev.tile == TC)
      (void)launch_k(k_pencil<0, 0, FX, TC>, grid, NT, pencil_smem_v(g), g->stream, g->dev, a);
    else
      (void)launch_k(k_pencil<0, 0, FX>, grid, NT, pencil_smem_v(g), g->stream, g->dev, a);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_pencil_to_cube_xmajor(pwb_grid* g, int nband, const double2* W, double scale,
                                 double2* out) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  PencilArgs a = empty_args();
  a.win = W;
  a.xin = g->dev.xa;
  a.nxin = g->nxa;
  a.in_stride = (size_t)g->nxa * g->nyz;
  a.mode = 2;
  a.cout = out;
  a.out_stride = (size_t)g->ng;
  a.oscale = scale;
  dim3 grid(tiles(g), nband);
  pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<0, 3, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_pencil_to_cube(pwb_grid* g, int nband, const double2* W, double scale, double2* out) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  PencilArgs a = empty_args();
  a.win = W;
  a.xin = g->dev.xa;
  a.nxin = g->nxa;
  a.in_stride = (size_t)g->nxa * g->nyz;
  a.mode = 2;
  a.cout = out;
  a.out_stride = (size_t)g->ng;
  a.oscale = scale;
  dim3 grid(tiles(g), nband);
  pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<0, 1, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_pencil_from_cube(pwb_grid* g, int nband, const double2* in, double2* W) {
  PWB_TRY(check_band_count(nband));
  if (nband == 0) return PWB_OK;
  PencilArgs a = empty_args();
  a.cin = in;
  a.in_stride = (size_t)g->ng;
  a.mode = 1;
  a.wout = W;
  a.xout = g->dev.xa;
  a.nxout = g->nxa;
  a.out_stride = (size_t)g->nxa * g->nyz;
  dim3 grid(tiles(g), nband);
  pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<1, 0, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_full_from_natural(pwb_grid* g, int nvec, const double2* in_c, const double* in_r,
                             int mode, double2* Wf) {
  PWB_TRY(check_band_count(nvec));
  if (nvec == 0) return PWB_OK;
  PencilArgs a = empty_args();
  a.cin = in_c;
  a.rin = in_r;
  a.in_stride = (size_t)g->ng;
  a.mode = mode;
  a.wout = Wf;
  a.xout = g->dev.xall;
  a.nxout = g->nx;
  a.out_stride = (size_t)g->ng;
  dim3 grid(tiles(g), nvec);
  if (in_c)
    pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<1, 0, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  else
    pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<2, 0, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_full_plane(pwb_grid* g, int nvec, double2* Wf, int mode, double param, int inverse) {
  PWB_TRY(check_band_count(nvec));
  if (nvec == 0) return PWB_OK;
  dim3 grid(g->nx, nvec);
  plane_variant(g, [&](auto fy, auto fz) {
    (void)launch_k(k_plane_full<decltype(fy), decltype(fz)>, grid, NT, plane_smem(g), g->stream, 
        g->dev, Wf, mode, param, inverse);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_full_to_natural(pwb_grid* g, int nvec, const double2* Wf, int mode, double scale,
                           double2* out_c, double* out_r, const double* v_lda,
                           const double* rho_lda) {
  PWB_TRY(check_band_count(nvec));
  if (nvec == 0) return PWB_OK;
  PencilArgs a = empty_args();
  a.win = Wf;
  a.xin = g->dev.xall;
  a.nxin = g->nx;
  a.in_stride = (size_t)g->ng;
  a.mode = mode;
  a.cout = out_c;
  a.rout = out_r;
  a.out_stride = (size_t)g->ng;
  a.oscale = scale;
  a.lda_v = v_lda;
  a.lda_rho = rho_lda;
  a.lda_c = -(1.0 / 3.0) * cbrt(3.0 / M_PI);
  dim3 grid(tiles(g), nvec);
  if (out_c)
    pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<0, 1, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  else
    pencil_variant(g, [&](auto fx) {
    (void)launch_k(k_pencil<0, 2, decltype(fx)>, grid, NT, pencil_smem(g), g->stream, g->dev, a);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int configure_kernels(const pwb_grid* g) {
  const size_t ps = plane_smem(g), cs = pencil_smem(g);
  if (ps > 227 * 1024 || pencil_smem_v(g) > 227 * 1024)
    return fail(PWB_ERR_UNSUPPORTED, "grid plane does not fit in shared memory");
  cudaError_t e = cudaSuccess;
  plane_variant(g, [&](auto fy, auto fz) {
    using FY = decltype(fy);
    using FZ = decltype(fz);
    e = cudaFuncSetAttribute(k_plane_inv<FY, FZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_plane_fwd<FY, FZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_plane_full<FY, FZ>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ps);
  });
  PWB_CUDA(e);
  pencil_variant(g, [&](auto fx) {
    using FX = decltype(fx);
    e = cudaFuncSetAttribute(k_pencil<0, 0, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pencil_smem_v(g));
    constexpr int TC = FX::N ? 3072 / FX::N : 0;
    if (e == cudaSuccess && TC)
      e = cudaFuncSetAttribute(k_pencil<0, 0, FX, TC ? TC : 1>,
                               cudaFuncAttributeMaxDynamicSharedMemorySize, (int)pencil_smem_v(g));
    if constexpr (TwoPass<FX::N>::ok) {
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_pencil_h<FX::N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pencil_smem_v(g));
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_pencil_hp<FX::N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)PencilHp<FX::N>::smem(g->nxa));
    }
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_pencil<0, 1, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_pencil<0, 3, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_pencil<0, 2, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_pencil<1, 0, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(k_pencil<2, 0, FX>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cs);
  });
  PWB_CUDA(e);
  return PWB_OK;
}

}  // namespace pwb
