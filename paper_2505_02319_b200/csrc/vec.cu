// Dense real-vector kernels for the device-resident inexact GMRES
// (reference igmres.py:86-114).  Dots use a fixed two-stage reduction
// (fixed grid, fixed order), so every scalar is bitwise reproducible; the
// MGS step keeps the Hessenberg entries on the device and returns the
// column to the host once per Arnoldi step.
#include <algorithm>
#include <cmath>

#include "grid.cuh"

namespace pwb {

constexpr int NTV = 256;
constexpr int kDotBlocks = 148;

__global__ void __launch_bounds__(NTV) k_dot_partial(int n, const double* __restrict__ x,
                                                     const double* __restrict__ y,
                                                     double* __restrict__ part) {
  pdl_wait();
  __shared__ double red[NTV];
  double s = 0.0;
  for (int i = blockIdx.x * NTV + threadIdx.x; i < n; i += gridDim.x * NTV) s += x[i] * y[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = NTV / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = red[0];
}

// out[0] = sum(part) (+= when accumulate), optional sqrt
__global__ void k_dot_final(int np, const double* __restrict__ part, double* __restrict__ out,
                            int accumulate, int take_sqrt) {
  pdl_wait();
  __shared__ double red[NTV];
  double s = 0.0;
  for (int i = threadIdx.x; i < np; i += NTV) s += part[i];
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = NTV / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    double v = red[0];
    if (take_sqrt) v = sqrt(v);
    out[0] = accumulate ? out[0] + v : v;
  }
}

// y -= c[0] * x   (c on device; sign flips via neg)
__global__ void k_axpy_dev(int n, const double* __restrict__ c, const double* __restrict__ x,
                           double* __restrict__ y) {
  pdl_wait();
  const double a = c[0];
  for (int i = blockIdx.x * NTV + threadIdx.x; i < n; i += gridDim.x * NTV) y[i] -= a * x[i];
}

__global__ void k_axpy_host(int n, double a, const double* __restrict__ x, double* __restrict__ y) {
  pdl_wait();
  for (int i = blockIdx.x * NTV + threadIdx.x; i < n; i += gridDim.x * NTV) y[i] += a * x[i];
}

// out = a x + b y (y == NULL: a x), each product and the sum rounded separately
// (no FMA contraction) so the result equals numpy's `a * x + b * y`
__global__ void k_axpby(long long n, double a, const double* __restrict__ x, double b,
                        const double* __restrict__ y, double* __restrict__ out) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)NTV + threadIdx.x; i < n;
       i += (long long)gridDim.x * NTV) {
    const double ax = __dmul_rn(a, x[i]);
    out[i] = y ? __dadd_rn(ax, __dmul_rn(b, y[i])) : ax;
  }
}

// out = x / d (IEEE division, numpy's `x / d`)
__global__ void k_div(long long n, const double* __restrict__ x, double d, double* __restrict__ out) {
  pdl_wait();
  for (long long i = blockIdx.x * (long long)NTV + threadIdx.x; i < n;
       i += (long long)gridDim.x * NTV)
    out[i] = __ddiv_rn(x[i], d);
}

// v = w / h (or 0 when h == 0: lucky breakdown, igmres.py:99-102)
__global__ void k_normalise(int n, const double* __restrict__ h, const double* __restrict__ w,
                            double* __restrict__ v) {
  pdl_wait();
  const double d = h[0];
  for (int i = blockIdx.x * NTV + threadIdx.x; i < n; i += gridDim.x * NTV)
    v[i] = d > 0.0 ? w[i] / d : 0.0;
}

// x = x0 + sum_j y_j V_j with the reference's sequential order
__global__ void k_combine(int n, int m, const double* __restrict__ V, const double* __restrict__ y,
                          const double* __restrict__ x0, double* __restrict__ x) {
  pdl_wait();
  for (int i = blockIdx.x * NTV + threadIdx.x; i < n; i += gridDim.x * NTV) {
    double s = x0[i];
    for (int j = 0; j < m; ++j) s = s + y[j] * V[(size_t)j * n + i];
    x[i] = s;
  }
}

// Grid-wide barrier for a launch whose CTAs are all co-resident (grid <= #SM,
// 256 threads, no smem): arrival counter + generation (bar zero-initialised
// once; the last arriver re-arms it).
__device__ __forceinline__ void grid_sync(unsigned* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    volatile unsigned* vb = bar;
    const unsigned gen = vb[1];
    __threadfence();
    if (atomicAdd(&bar[0], 1u) == gridDim.x - 1) {
      bar[0] = 0u;
      __threadfence();
      atomicAdd(&bar[1], 1u);
    } else {
      while (vb[1] == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// sum of this launch's per-CTA partials, fixed order, identical on every CTA
__device__ __forceinline__ double grid_sum(const double* part, double* red) {
  double s = 0.0;
  for (int b = threadIdx.x; b < (int)gridDim.x; b += NTV) s += __ldcg(&part[b]);
  red[threadIdx.x] = s;
  __syncthreads();
  for (int o = NTV / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  const double v = red[0];
  __syncthreads();
  return v;
}

// One Arnoldi step's modified Gram-Schmidt with one re-orthogonalisation
// (igmres.py:86-103) as ONE launch: per projection, CTA partial dots -> grid
// barrier -> every CTA sums the partials in the same order and updates its own
// slice of w (the slice mapping is the same for dot and update, so no other
// cross-CTA dependency).  2 (i + 1) + 1 barriers instead of 6 (i + 1) + 3
// launches; hd as in pwb_arnoldi_mgs ([0..i] pass 1, [i+1..2i+1] pass 2, norm).
__global__ void __launch_bounds__(NTV) k_mgs_fused(int n, int i, const double* __restrict__ V,
                                                   double* __restrict__ w,
                                                   double* __restrict__ vnext,
                                                   double* __restrict__ part,
                                                   double* __restrict__ hd,
                                                   unsigned* __restrict__ bar) {
  pdl_wait();
  __shared__ double red[NTV];
  const int nb = gridDim.x;
  const int i0 = blockIdx.x * NTV + threadIdx.x, st = gridDim.x * NTV;
  for (int q = 0; q < 2 * (i + 1) + 1; ++q) {
    const bool norm = q == 2 * (i + 1);
    const double* vj = norm ? w : V + (size_t)(q % (i + 1)) * n;
    double acc = 0.0;
    for (int e = i0; e < n; e += st) acc += vj[e] * w[e];
    red[threadIdx.x] = acc;
    __syncthreads();
    for (int o = NTV / 2; o > 0; o >>= 1) {
      if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
      __syncthreads();
    }
    if (threadIdx.x == 0) part[(size_t)q * nb + blockIdx.x] = red[0];
    grid_sync(bar);
    const double h = grid_sum(part + (size_t)q * nb, red);
    if (!norm) {
      for (int e = i0; e < n; e += st) w[e] -= h * vj[e];
      if (blockIdx.x == 0 && threadIdx.x == 0) hd[q] = h;
    } else {
      const double d = sqrt(h);
      for (int e = i0; e < n; e += st) vnext[e] = d > 0.0 ? w[e] / d : 0.0;
      if (blockIdx.x == 0 && threadIdx.x == 0) hd[q] = d;
    }
  }
}

// vector ops may run without a grid (generic GMRES use): default stream and
// thread-local scratch
struct VecCtx {
  cudaStream_t stream;
  DevBuf* red;
  DevBuf* scratch;
};

static VecCtx vctx(pwb_grid* g) {
  static thread_local DevBuf red, scratch;
  if (g) return VecCtx{g->stream, &g->red, &g->scratch};
  return VecCtx{nullptr, &red, &scratch};
}

static int blocks_for(int n) { return std::max(1, std::min(kDotBlocks, (n + NTV - 1) / NTV)); }

static int dot_into(const VecCtx& c, int n, const double* x, const double* y, double* out,
                    int accumulate, int take_sqrt) {
  PWB_TRY(c.red->ensure(kDotBlocks * sizeof(double)));
  const int nb = blocks_for(n);
  (void)launch_k(k_dot_partial, nb, NTV, 0, c.stream, n, x, y, as<double>(*c.red));
  PWB_LAUNCH_CHECK();
  (void)launch_k(k_dot_final, 1, NTV, 0, c.stream, nb, as<double>(*c.red), out, accumulate, take_sqrt);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

}  // namespace pwb

using namespace pwb;

extern "C" {

int pwb_vec_dot(pwb_grid* g, int n, const double* x, const double* y, double* out_dev) {
  return dot_into(vctx(g), n, x, y, out_dev, 0, 0);
}

int pwb_vec_axpby(pwb_grid* g, long long n, double a, const double* x, double b, const double* y,
                  double* out) {
  if (n <= 0) return PWB_OK;
  if (!x || !out) return fail(PWB_ERR_VALUE, "null vector");
  const int nb = (int)std::min<long long>(4LL * kSM, (n + NTV - 1) / NTV);
  (void)launch_k(k_axpby, nb, NTV, 0, vctx(g).stream, n, a, x, b, y, out);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int pwb_vec_div(pwb_grid* g, long long n, const double* x, double d, double* out) {
  if (n <= 0) return PWB_OK;
  if (!x || !out) return fail(PWB_ERR_VALUE, "null vector");
  const int nb = (int)std::min<long long>(4LL * kSM, (n + NTV - 1) / NTV);
  (void)launch_k(k_div, nb, NTV, 0, vctx(g).stream, n, x, d, out);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int pwb_vec_axpy(pwb_grid* g, int n, double a, const double* x, double* y) {
  (void)launch_k(k_axpy_host, blocks_for(n), NTV, 0, vctx(g).stream, n, a, x, y);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int pwb_arnoldi_mgs(pwb_grid* g, int n, int i, double* basis, double* w, double* hcol_host) {
  if (i < 0) return fail(PWB_ERR_VALUE, "negative Arnoldi index");
  const VecCtx c = vctx(g);
  PWB_TRY(c.scratch->ensure((size_t)(2 * (i + 1) + 1) * sizeof(double)));
  double* hd = as<double>(*c.scratch);   // [0..i]: pass 1, [i+1..2i+1]: pass 2, [2i+2]: norm
  const int nb = blocks_for(n);
  static const bool no_fused = getenv("PWB_NO_FUSED_MGS") != nullptr;   // A/B measurement
  bool fused = !no_fused && g;
  if (fused) {
    PWB_TRY(g->mgs_part.ensure((size_t)(2 * (i + 1) + 1) * kDotBlocks * sizeof(double)));
    if (!g->mgs_bar.ptr) {
      PWB_TRY(g->mgs_bar.ensure(2 * sizeof(unsigned)));
      PWB_CUDA(cudaMemset(g->mgs_bar.ptr, 0, 2 * sizeof(unsigned)));
    }
    // the grid barrier needs every CTA resident: cooperative launch, which fails
    // (instead of hanging) when SM partitioning / concurrent kernels prevent it;
    // then the unfused dot / axpy sequence below runs instead
    const cudaError_t e = launch_coop(k_mgs_fused, nb, NTV, 0, c.stream, n, i,
                                      (const double*)basis, w, basis + (size_t)(i + 1) * n,
                                      as<double>(g->mgs_part), hd, as<unsigned>(g->mgs_bar));
    if (e != cudaSuccess) {
      (void)cudaGetLastError();
      fused = false;
    } else {
      count_launch();
    }
  }
  if (!fused) {
  for (int pass = 0; pass < 2; ++pass)
    for (int j = 0; j <= i; ++j) {
      double* c = hd + pass * (i + 1) + j;
      PWB_TRY(dot_into(vctx(g), n, basis + (size_t)j * n, w, c, 0, 0));
      (void)launch_k(k_axpy_dev, nb, NTV, 0, vctx(g).stream, n, c, basis + (size_t)j * n, w);
      PWB_LAUNCH_CHECK();
    }
  double* nrm = hd + 2 * (i + 1);
  PWB_TRY(dot_into(c, n, w, w, nrm, 0, 1));
  (void)launch_k(k_normalise, nb, NTV, 0, c.stream, n, nrm, w, basis + (size_t)(i + 1) * n);
  PWB_LAUNCH_CHECK();
  }
  std::vector<double> hh(2 * (i + 1) + 1);
  PWB_CUDA(cudaMemcpyAsync(hh.data(), hd, hh.size() * sizeof(double), cudaMemcpyDeviceToHost,
                           c.stream));
  PWB_CUDA(cudaStreamSynchronize(c.stream));
  for (int j = 0; j <= i; ++j) hcol_host[j] = hh[j] + hh[i + 1 + j];
  hcol_host[i + 1] = hh[2 * (i + 1)];
  return PWB_OK;
}

int pwb_vec_combine(pwb_grid* g, int n, int m, const double* basis, const double* y_host,
                    const double* x0, double* x) {
  const VecCtx c = vctx(g);
  PWB_TRY(c.scratch->ensure((size_t)std::max(m, 1) * sizeof(double)));
  if (m > 0)
    PWB_CUDA(cudaMemcpyAsync(c.scratch->ptr, y_host, m * sizeof(double), cudaMemcpyHostToDevice,
                             c.stream));
  (void)launch_k(k_combine, blocks_for(n), NTV, 0, c.stream, n, m, basis, as<double>(*c.scratch), x0, x);
  PWB_LAUNCH_CHECK();
  PWB_CUDA(cudaStreamSynchronize(c.stream));
  return PWB_OK;
}

}  // extern "C"
