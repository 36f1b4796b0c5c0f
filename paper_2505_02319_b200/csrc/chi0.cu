// Density-response accumulation (reference response.py:150-154):
//   drho(r) = sum_b [ c2_b Re(conj psi_b(r) dphi~_b(r)) + c1_b |psi_b(r)|^2 ]
// with dphi~_b the unnormalised inverse transform of the orbital response
// (c2_b = w_k 2 f_n / sqrt(Omega) carries the to_real scale) and psi_b(r)
// from the per-state cache.  The inverse x-FFT of dphi is fused into the
// accumulation, so dphi(r) never reaches HBM; bands are reduced in a fixed
// order inside each CTA and chunk partials are summed in a fixed order, so
// drho is bitwise reproducible (no floating-point atomics).
#include "dispatch.cuh"
#include "state.cuh"

namespace pwb {

constexpr int NTA = 256;
constexpr int kMaxOwn = 16;   // tile elements per thread (tile*nx <= 3072 + pad)

template <class FX>
__global__ void __launch_bounds__(NTA) k_drho_partial(GridDev g, int nband, int per_chunk,
                                                      const double2* __restrict__ W,
                                                      const double2* __restrict__ psir,
                                                      const double* __restrict__ c2,
                                                      const double* __restrict__ c1,
                                                      double* __restrict__ partial) {
  pdl_wait();
  extern __shared__ double2 sm[];
  const int T = g.tile, Tp = g.tilep, nx = g.nx, nyz = g.nyz;
  const int t0 = blockIdx.x * T;
  const int nt = min(T, nyz - t0);
  const int b0 = blockIdx.y * per_chunk;
  const int b1 = min(nband, b0 + per_chunk);
  const int nel = nt * nx;
  double acc[kMaxOwn];
#pragma unroll
  for (int q = 0; q < kMaxOwn; ++q) acc[q] = 0.0;
  for (int b = b0; b < b1; ++b) {
    for (int i = threadIdx.x; i < nx * Tp; i += NTA) sm[i] = make_double2(0.0, 0.0);
    __syncthreads();
    const double2* src = W + (size_t)b * g.nxa * nyz;
    staged_copy<6, NTA>(
        g.nxa * nt,
        [&](int i) {
          const int p = i / nt;
          return __ldg(&src[(size_t)p * nyz + t0 + (i - p * nt)]);
        },
        [&](int i, double2 v) {
          const int p = i / nt;
          sm[g.xa[p] * Tp + (i - p * nt)] = v;
        });
    __syncthreads();
    FX::template run<NTA>(g, sm, nt, Tp, 1, nullptr, true);
    const double a2 = c2[b], a1 = c1[b];
    const double2* ps = psir + (size_t)b * g.ng + t0;   // x-major cache [x][yz]
#pragma unroll
    for (int q = 0; q < kMaxOwn; ++q) {
      const int i = threadIdx.x + q * NTA;
      if (i < nel) {
        const int t = i / nx, x = i - t * nx;
        const double2 d = sm[x * Tp + t];
        const double2 p = ps[(size_t)x * nyz + t];
        acc[q] += a2 * (p.x * d.x + p.y * d.y) + a1 * (p.x * p.x + p.y * p.y);
      }
    }
    __syncthreads();
  }
  double* out = partial + (size_t)blockIdx.y * g.ng + (size_t)t0 * nx;
#pragma unroll
  for (int q = 0; q < kMaxOwn; ++q) {
    const int i = threadIdx.x + q * NTA;
    if (i < nel) out[i] = acc[q];
  }
}

// Two-pass lengths (TwoPass<N>, fft_kernels.cu): per band the inverse x-FFT
// runs as pass A (radix R1, W rows straight from global, active x only) ->
// smem -> pass B (radix R2, natural-order outputs in registers), and pass B's
// outputs are accumulated directly against the x-major psi(r) cache: two
// barriers per band instead of eight, no smem zero-fill, coalesced psi loads.
// Each thread owns the same (x, column) elements for every band, so the band
// sum is in fixed order (bitwise reproducible).
template <int N>
__global__ void __launch_bounds__(NTA, 3) k_drho_h(GridDev g, int nband, int per_chunk,
                                                   const double2* __restrict__ W,
                                                   const double2* __restrict__ psir,
                                                   const double* __restrict__ c2,
                                                   const double* __restrict__ c1,
                                                   double* __restrict__ partial) {
  constexpr int R1 = TwoPass<N>::R1, R2 = TwoPass<N>::R2;
  constexpr int TC = 3072 / N, TP = (TC % 2 == 0) ? TC + 1 : TC;
  constexpr int NB1 = N / R1, LP1 = NTA / NB1, LP2 = NTA / R1;
  constexpr int MB = (TC + LP2 - 1) / LP2;
  pdl_wait();
  extern __shared__ double2 sm[];
  const int nyz = g.nyz;
  const int t0 = blockIdx.x * TC;
  const int nt = min(TC, nyz - t0);
  const int b0 = blockIdx.y * per_chunk;
  const int b1 = min(nband, b0 + per_chunk);
  const int x0 = g.xa[0], nxa = g.nxa;
  const int tid = threadIdx.x;
  const int ja = tid / LP1, la = tid - ja * LP1;   // pass A: butterfly ja of lines la, la + LP1..
  const int jb = tid / LP2, lb = tid - jb * LP2;   // pass B: butterfly jb of lines lb + m LP2
  constexpr bool kHoldW = R2 <= 8;   // radix 12: twiddles from L1 per use (registers)
  double2 w[kHoldW ? R2 : 1];
  if constexpr (kHoldW) {
#pragma unroll
    for (int r = 1; r < R2; ++r) {
      const double2 t = __ldg(&g.px.tw[r * jb]);
      w[r] = make_double2(t.x, -t.y);   // inverse
    }
  }
  double acc[MB][R2];
#pragma unroll
  for (int m = 0; m < MB; ++m)
#pragma unroll
    for (int r = 0; r < R2; ++r) acc[m][r] = 0.0;
  for (int b = b0; b < b1; ++b) {
    const double2* src = W + (size_t)b * nxa * nyz;
    if (ja < NB1) {
      for (int l = la; l < TC; l += LP1) {
        double2 v[R1];
#pragma unroll
        for (int r = 0; r < R1; ++r) {
          int p = ja + r * NB1 - x0;
          if (p < 0) p += N;
          v[r] = (p < nxa && l < nt) ? __ldg(&src[(size_t)p * nyz + t0 + l])
                                     : make_double2(0.0, 0.0);
        }
        Dft<R1>::run(v, 1.0);
#pragma unroll
        for (int r = 0; r < R1; ++r) sm[(ja * R1 + r) * TP + l] = v[r];
      }
    }
    __syncthreads();
    const double a2 = c2[b], a1 = c1[b];
    const double2* ps = psir + (size_t)b * g.ng + t0;
#pragma unroll
    for (int m = 0; m < MB; ++m) {
      const int l = m * LP2 + lb;
      if (l < nt) {
        double2 v[R2], p[R2];
#pragma unroll
        for (int r = 0; r < R2; ++r) {
          v[r] = sm[(jb + r * R1) * TP + l];
          p[r] = __ldg(&ps[(size_t)(jb + r * R1) * nyz + l]);
        }
#pragma unroll
        for (int r = 1; r < R2; ++r) {
          if constexpr (kHoldW) {
            v[r] = cmul(v[r], w[r]);
          } else {
            const double2 t = __ldg(&g.px.tw[r * jb]);
            v[r] = cmul(v[r], make_double2(t.x, -t.y));
          }
        }
        Dft<R2>::run(v, 1.0);   // outputs x = jb + r R1 (natural order)
#pragma unroll
        for (int r = 0; r < R2; ++r)
          acc[m][r] += a2 * (p[r].x * v[r].x + p[r].y * v[r].y) +
                       a1 * (p[r].x * p[r].x + p[r].y * p[r].y);
      }
    }
    __syncthreads();   // the next band's pass A overwrites smem
  }
  double* out = partial + (size_t)blockIdx.y * g.ng + (size_t)t0 * N;
#pragma unroll
  for (int m = 0; m < MB; ++m) {
    const int l = m * LP2 + lb;
    if (l < nt) {
#pragma unroll
      for (int r = 0; r < R2; ++r) out[(size_t)l * N + jb + r * R1] = acc[m][r];
    }
  }
}

__global__ void k_drho_reduce(int n, int nchunk, const double* __restrict__ partial,
                              double* __restrict__ drho) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = partial[i];
  for (int c = 1; c < nchunk; ++c) s += partial[(size_t)c * n + i];
  drho[i] = s;
}

// out[i] = sum_b |psi_b(i)|^2  (or (Re psi_b)^2); max taken by k_max_reduce
__global__ void k_row_sq(int n, int nband, const double2* __restrict__ psir, int real_part,
                         double* __restrict__ out) {
  pdl_wait();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double s = 0.0;
  for (int b = 0; b < nband; ++b) {
    const double2 p = psir[(size_t)b * n + i];
    s += real_part ? p.x * p.x : p.x * p.x + p.y * p.y;
  }
  out[i] = s;
}

__global__ void k_max_reduce(int n, const double* __restrict__ in, double* __restrict__ out) {
  pdl_wait();
  __shared__ double red[256];
  double m = 0.0;
  for (int i = threadIdx.x; i < n; i += 256) m = fmax(m, in[i]);
  red[threadIdx.x] = m;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] = fmax(red[threadIdx.x], red[threadIdx.x + s]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = red[0];
}

int launch_drho_partial(pwb_grid* g, int nband, const double2* W, const double2* psir,
                        const double* c2, const double* c1, int nchunk, double* partial) {
  if (g->dev.tile * g->nx > kMaxOwn * NTA)
    return fail(PWB_ERR_UNSUPPORTED, "pencil tile too large for accumulation kernel");
  const int ntile = (g->nyz + g->dev.tile - 1) / g->dev.tile;
  const int per = (nband + nchunk - 1) / nchunk;
  dim3 grid(ntile, nchunk);
  static const bool generic_only = getenv("PWB_NO_PENCIL_H") != nullptr;   // A/B measurement
  pencil_variant(g, [&](auto fx) {
    using FX = decltype(fx);
    if constexpr (TwoPass<FX::N>::ok) {
      if (!generic_only && g->dev.tile == 3072 / FX::N) {
        (void)launch_k(k_drho_h<FX::N>, grid, NTA, pencil_smem(g), g->stream, g->dev, nband, per,
                       W, psir, c2, c1, partial);
        return;
      }
    }
    (void)launch_k(k_drho_partial<FX>, grid, NTA, pencil_smem(g), g->stream, g->dev, nband, per,
                   W, psir, c2, c1, partial);
  });
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_drho_reduce(pwb_grid* g, int nchunk, const double* partial, double* drho) {
  (void)launch_k(k_drho_reduce, (g->ng + 255) / 256, 256, 0, g->stream, g->ng, nchunk, partial, drho);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int launch_row_norm(pwb_grid* g, int nband, const double2* psir, int real_part, double* out) {
  PWB_TRY(g->tmp_real.ensure((size_t)(g->ng + 1) * sizeof(double)));
  double* sq = as<double>(g->tmp_real);
  (void)launch_k(k_row_sq, (g->ng + 255) / 256, 256, 0, g->stream, g->ng, nband, psir, real_part, sq);
  PWB_LAUNCH_CHECK();
  (void)launch_k(k_max_reduce, 1, 256, 0, g->stream, g->ng, sq, out);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int configure_chi0_kernels(const pwb_grid* g) {
  cudaError_t e = cudaSuccess;
  pencil_variant(g, [&](auto fx) {
    using FX = decltype(fx);
    e = cudaFuncSetAttribute(k_drho_partial<FX>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             (int)pencil_smem(g));
    if constexpr (TwoPass<FX::N>::ok) {
      if (e == cudaSuccess)
        e = cudaFuncSetAttribute(k_drho_h<FX::N>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 (int)pencil_smem(g));
    }
  });
  PWB_CUDA(e);
  return PWB_OK;
}

}  // namespace pwb
