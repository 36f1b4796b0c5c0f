// Occupied-subspace projector Q = 1 - Phi Phi^H as two complex-FP64 GEMMs on
// the FP64 tensor pipe (DMMA: mma.sync.m8n8k4.f64), reference
// sternheimer.py:28-30 and response.py:129,138.
//
//   coef :  C[row][m] = sum_g conj(Phi_k[m][g]) X[row][g]
//           split-K over the sphere (grid covers the 148 SMs); warps of a CTA
//           reduce in smem, CTAs reduce through a partial buffer in FIXED
//           split order by the last CTA to finish (threadfence + counter):
//           bitwise reproducible, one launch.
//   apply:  Y[row][g] = a X[row][g] + b sum_m Phi_k[m][g] C[row][m]
//
// Complex products are four real DMMAs (re.re, im.im, re.im, im.re).  Rows of
// X are grouped in tiles of <= 16 rows sharing one k block; with active-row
// compaction the tile rows index X through a row list.
// Measured on B200: DMMA 37.1 TFLOP/s, DFMA 34.0 TFLOP/s (tools/fp64_peak.cu).
#include "proj.cuh"

namespace pwb {

constexpr int TR = 16;   // rows per tile (2 DMMA n-fragments)
constexpr int CM = 32;   // m per coef block (4 DMMA m-fragments)
constexpr int CW = 4;    // warps per CTA
constexpr int AG = 128;  // g per apply CTA (4 warps x 32)

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

__device__ __forceinline__ int xrow(const ProjArgs& a, const ProjTile& t, int r) {
  return a.rows ? a.rows[t.row0 + r] : t.row0 + r;
}

// grid (tiles, m blocks, splits), 128 threads
__global__ void __launch_bounds__(CW * 32) k_proj_coef(ProjArgs a, const double2* __restrict__ X,
                                                       int split_len, int nsplit,
                                                       double2* __restrict__ part,
                                                       double2* __restrict__ C,
                                                       unsigned* __restrict__ counters) {
  __shared__ double2 red[CW][CM][TR];
  __shared__ bool last;
  const ProjTile t = a.tiles[blockIdx.x];
  const int m0 = blockIdx.y * CM;
  const int nocc = a.nocc[t.k];
  if (m0 >= nocc) return;
  const int split = blockIdx.z;
  const int g0 = split * split_len;
  const int g1 = min(a.nbp, g0 + split_len);
  const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  // fragment source rows
  const double2* prow[4];
  bool pok[4];
#pragma unroll
  for (int ma = 0; ma < 4; ++ma) {
    const int m = m0 + 8 * ma + r4;
    pok[ma] = m < nocc;
    prow[ma] = phi + (size_t)(pok[ma] ? m : 0) * a.nbp;
  }
  const double2* xrw[2];
  bool xok[2];
#pragma unroll
  for (int nb = 0; nb < 2; ++nb) {
    const int r = 8 * nb + r4;
    xok[nb] = r < t.nrows;
    xrw[nb] = X + (size_t)(xok[nb] ? xrow(a, t, r) : 0) * a.nbp;
  }
  double cr[4][2][2], ci[4][2][2];
#pragma unroll
  for (int ma = 0; ma < 4; ++ma)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      cr[ma][nb][0] = cr[ma][nb][1] = 0.0;
      ci[ma][nb][0] = ci[ma][nb][1] = 0.0;
    }
  for (int g = g0 + 4 * w; g < g1; g += 4 * CW) {
    const int gg = g + c4;
    const bool gok = gg < g1;
    double2 av[4], bv[2];
#pragma unroll
    for (int ma = 0; ma < 4; ++ma)
      av[ma] = (gok && pok[ma]) ? __ldg(&prow[ma][gg]) : make_double2(0.0, 0.0);
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
      bv[nb] = (gok && xok[nb]) ? xrw[nb][gg] : make_double2(0.0, 0.0);
#pragma unroll
    for (int ma = 0; ma < 4; ++ma)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        // conj(phi) * x : re = pr xr + pi xi ; im = pr xi - pi xr
        dmma(cr[ma][nb][0], cr[ma][nb][1], av[ma].x, bv[nb].x);
        dmma(cr[ma][nb][0], cr[ma][nb][1], av[ma].y, bv[nb].y);
        dmma(ci[ma][nb][0], ci[ma][nb][1], av[ma].x, bv[nb].y);
        dmma(ci[ma][nb][0], ci[ma][nb][1], -av[ma].y, bv[nb].x);
      }
  }
  // D fragment: (m = r4, row = 2 c4 + {0,1}) of each (ma, nb) tile
#pragma unroll
  for (int ma = 0; ma < 4; ++ma)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int h = 0; h < 2; ++h)
        red[w][8 * ma + r4][8 * nb + 2 * c4 + h] = make_double2(cr[ma][nb][h], ci[ma][nb][h]);
  __syncthreads();
  // fixed-order sum over warps -> this split's partial
  const size_t tile_id = (size_t)blockIdx.x * gridDim.y + blockIdx.y;
  double2* mypart = part + ((size_t)split * gridDim.x * gridDim.y + tile_id) * (CM * TR);
  for (int i = threadIdx.x; i < CM * TR; i += CW * 32) {
    const int m = i / TR, r = i - m * TR;
    double2 s = red[0][m][r];
#pragma unroll
    for (int q = 1; q < CW; ++q) s = cadd(s, red[q][m][r]);
    if (nsplit == 1) {
      if (r < t.nrows && m0 + m < nocc) C[(size_t)(t.row0 + r) * a.ldc + m0 + m] = s;
    } else {
      mypart[i] = s;
    }
  }
  if (nsplit == 1) return;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(&counters[tile_id], 1u);
    last = (prev == (unsigned)nsplit - 1);
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  const size_t stride = (size_t)gridDim.x * gridDim.y * (CM * TR);
  const double2* p0 = part + tile_id * (CM * TR);
  for (int i = threadIdx.x; i < CM * TR; i += CW * 32) {
    const int m = i / TR, r = i - m * TR;
    double2 s = p0[i];
    for (int q = 1; q < nsplit; ++q) s = cadd(s, p0[(size_t)q * stride + i]);
    if (r < t.nrows && m0 + m < nocc) C[(size_t)(t.row0 + r) * a.ldc + m0 + m] = s;
  }
  if (threadIdx.x == 0) counters[tile_id] = 0u;
}

// grid (tiles, g chunks of 128), 128 threads; warp w covers g0 + 32 w .. + 32
__global__ void __launch_bounds__(CW * 32) k_proj_apply(ProjArgs a, const double2* __restrict__ C,
                                                        const double2* __restrict__ Xin,
                                                        double2* __restrict__ Y, double ca,
                                                        double cb, const int* __restrict__ active,
                                                        int band_mod) {
  const ProjTile t = a.tiles[blockIdx.x];
  const int nocc = a.nocc[t.k];
  const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  const int gw = blockIdx.y * AG + 32 * w;
  double dr[2][4][2], di[2][4][2];
#pragma unroll
  for (int jb = 0; jb < 2; ++jb)
#pragma unroll
    for (int gb = 0; gb < 4; ++gb) {
      dr[jb][gb][0] = dr[jb][gb][1] = 0.0;
      di[jb][gb][0] = di[jb][gb][1] = 0.0;
    }
  if (gw < a.nbp) {
    for (int m = 0; m < nocc; m += 4) {
      const int mm = m + c4;
      const bool mok = mm < nocc;
      double2 av[2], bv[4];
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        const int r = 8 * jb + r4;   // A[j = r4][k = c4] = C[row j][m + c4]
        av[jb] = (mok && r < t.nrows) ? C[(size_t)(t.row0 + r) * a.ldc + mm]
                                      : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int gb = 0; gb < 4; ++gb) {
        const int g = gw + 8 * gb + r4;   // B[k = c4][n = r4] = Phi[m + c4][g]
        bv[gb] = (mok && g < a.nbp) ? __ldg(&phi[(size_t)mm * a.nbp + g]) : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int jb = 0; jb < 2; ++jb)
#pragma unroll
        for (int gb = 0; gb < 4; ++gb) {
          // C * Phi : re = cr pr - ci pi ; im = cr pi + ci pr
          dmma(dr[jb][gb][0], dr[jb][gb][1], av[jb].x, bv[gb].x);
          dmma(dr[jb][gb][0], dr[jb][gb][1], -av[jb].y, bv[gb].y);
          dmma(di[jb][gb][0], di[jb][gb][1], av[jb].x, bv[gb].y);
          dmma(di[jb][gb][0], di[jb][gb][1], av[jb].y, bv[gb].x);
        }
    }
  }
  // D fragment: row j = r4, g = 2 c4 + {0,1}
#pragma unroll
  for (int jb = 0; jb < 2; ++jb) {
    const int r = 8 * jb + r4;
    if (r >= t.nrows) continue;
    const int row = a.rows ? a.rows[t.row0 + r] : t.row0 + r;
    if (active && !active[row % band_mod]) continue;
#pragma unroll
    for (int gb = 0; gb < 4; ++gb)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int g = gw + 8 * gb + 2 * c4 + h;
        if (g >= a.nbp) continue;
        const size_t idx = (size_t)row * a.nbp + g;
        const double2 x = (ca != 0.0) ? Xin[idx] : make_double2(0.0, 0.0);
        Y[idx] = make_double2(ca * x.x + cb * dr[jb][gb][h], ca * x.y + cb * di[jb][gb][h]);
      }
  }
}

int proj_plan(ProjPlan& pl, const std::vector<int>& row_k, const std::vector<int>& nocc,
              int nbp) {
  pl.tiles.clear();
  const int n = (int)row_k.size();
  int i = 0;
  int maxocc = 0;
  while (i < n) {
    int j = i;
    while (j < n && row_k[j] == row_k[i] && j - i < TR) ++j;
    pl.tiles.push_back(ProjTile{i, j - i, row_k[i]});
    maxocc = std::max(maxocc, nocc[row_k[i]]);
    i = j;
  }
  pl.nrows = n;
  pl.mtiles = (maxocc + CM - 1) / CM;
  const int ntiles = (int)pl.tiles.size();
  const int base = std::max(1, ntiles * pl.mtiles);
  int want = (2 * kSM + base - 1) / base;
  const int maxsplit = std::max(1, nbp / (16 * CW));
  pl.nsplit = std::min(std::max(1, want), maxsplit);
  int len = (nbp + pl.nsplit - 1) / pl.nsplit;
  len = ((len + 4 * CW - 1) / (4 * CW)) * (4 * CW);
  pl.split_len = len;
  pl.nsplit = (nbp + len - 1) / len;
  PWB_TRY(pl.dtiles.ensure(std::max<size_t>(1, pl.tiles.size()) * sizeof(ProjTile)));
  if (!pl.tiles.empty())
    PWB_CUDA(cudaMemcpy(pl.dtiles.ptr, pl.tiles.data(), pl.tiles.size() * sizeof(ProjTile),
                        cudaMemcpyHostToDevice));
  const size_t ntm = (size_t)ntiles * pl.mtiles;
  if (pl.counters.bytes < ntm * sizeof(unsigned) || !pl.counters.ptr) {
    PWB_TRY(pl.counters.ensure(std::max<size_t>(1, ntm) * sizeof(unsigned)));
    PWB_CUDA(cudaMemset(pl.counters.ptr, 0, std::max<size_t>(1, ntm) * sizeof(unsigned)));
  }
  return PWB_OK;
}

size_t proj_part_elems(const ProjPlan& pl) {
  return (size_t)pl.nsplit * pl.tiles.size() * pl.mtiles * CM * TR;
}

int proj_coeffs(const ProjPlan& pl, ProjArgs a, const double2* X, double2* part, double2* C,
                cudaStream_t st) {
  if (pl.tiles.empty()) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  dim3 grid((unsigned)pl.tiles.size(), pl.mtiles, pl.nsplit);
  k_proj_coef<<<grid, CW * 32, 0, st>>>(a, X, pl.split_len, pl.nsplit, part, C,
                                        reinterpret_cast<unsigned*>(pl.counters.ptr));
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int proj_apply(const ProjPlan& pl, ProjArgs a, const double2* C, const double2* Xin, double2* Y,
               double ca, double cb, const int* active, int band_mod, cudaStream_t st) {
  if (pl.tiles.empty()) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  dim3 grid((unsigned)pl.tiles.size(), (a.nbp + AG - 1) / AG);
  k_proj_apply<<<grid, CW * 32, 0, st>>>(a, C, Xin, Y, ca, cb, active, band_mod > 0 ? band_mod : 1);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

}  // namespace pwb
