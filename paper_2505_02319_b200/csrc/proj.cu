// Occupied-subspace projector Q = 1 - Phi Phi^H as two complex-FP64 GEMMs
// (reference: sternheimer.py:28-30, response.py:129,138).
//
//   partial:  C_s[row][m] = sum_{g in split s} conj(Phi_k[m][g]) X[row][g]
//   reduce :  C[row][m]   = sum_s C_s[row][m]          (fixed split order)
//   apply  :  Y[row][g]   = a X[row][g] + b sum_m Phi_k[m][g] C[row][m]
//
// Rows of X are grouped in tiles of <= 32 consecutive rows sharing one
// k block.  The contraction dimension (the padded sphere, up to ~16k for
// config 4) is split so the grid covers the 148 SMs; the split partials are
// reduced in a fixed order, so results are bitwise reproducible.
#include "proj.cuh"

namespace pwb {

constexpr int TR = 32;      // rows per tile
constexpr int TM = 32;      // m per tile (partial)
constexpr int TS = 32;      // g sub-chunk (partial)
constexpr int AS = 64;      // g chunk (apply)

// 64 threads, 4x4 (rows x m) per thread.
__global__ void __launch_bounds__(64) k_proj_partial(ProjArgs a, const double2* __restrict__ X,
                                                     int split_len, double2* __restrict__ part) {
  __shared__ double2 xs[TR][TS + 1];
  __shared__ double2 ps[TM][TS + 1];
  const ProjTile t = a.tiles[blockIdx.x];
  const int m0 = blockIdx.y * TM;
  const int nocc = a.nocc[t.k];
  if (m0 >= nocc) return;
  const int split = blockIdx.z;
  const int g0 = split * split_len;
  const int g1 = min(a.nbp, g0 + split_len);
  const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
  const int tr = threadIdx.x & 7, tm = threadIdx.x >> 3;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);

  for (int gs = g0; gs < g1; gs += TS) {
    const int len = min(TS, g1 - gs);
    for (int e = threadIdx.x; e < TR * TS; e += 64) {
      const int r = e / TS, c = e - r * TS;
      double2 xv = make_double2(0.0, 0.0), pv = make_double2(0.0, 0.0);
      if (c < len) {
        if (r < t.nrows) xv = X[(size_t)(t.row0 + r) * a.nbp + gs + c];
        if (m0 + r < nocc) pv = phi[(size_t)(m0 + r) * a.nbp + gs + c];
      }
      xs[r][c] = xv;
      ps[r][c] = pv;
    }
    __syncthreads();
#pragma unroll 4
    for (int c = 0; c < TS; ++c) {
      double2 xv[4], pv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) xv[i] = xs[tr + 8 * i][c];
#pragma unroll
      for (int j = 0; j < 4; ++j) pv[j] = ps[tm + 8 * j][c];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          // conj(p) * x
          acc[i][j].x = fma(pv[j].x, xv[i].x, acc[i][j].x);
          acc[i][j].x = fma(pv[j].y, xv[i].y, acc[i][j].x);
          acc[i][j].y = fma(pv[j].x, xv[i].y, acc[i][j].y);
          acc[i][j].y = fma(-pv[j].y, xv[i].x, acc[i][j].y);
        }
    }
    __syncthreads();
  }
  double2* out = part + (size_t)split * a.nrows_total * a.ldc;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = tr + 8 * i;
    if (r >= t.nrows) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int m = m0 + tm + 8 * j;
      if (m < nocc) out[(size_t)(t.row0 + r) * a.ldc + m] = acc[i][j];
    }
  }
}

// C[row][m] = sum_s part[s][row][m], fixed order.
__global__ void k_proj_reduce(int nsplit, size_t n, const double2* __restrict__ part,
                              double2* __restrict__ C) {
  const size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double2 s = part[i];
  for (int q = 1; q < nsplit; ++q) s = cadd(s, part[(size_t)q * n + i]);
  C[i] = s;
}

// 128 threads, tile 32 rows x 64 g, 4x4 (rows x g) per thread.
__global__ void __launch_bounds__(128) k_proj_apply(ProjArgs a, const double2* __restrict__ C,
                                                    const double2* __restrict__ Xin,
                                                    double2* __restrict__ Y, double ca, double cb,
                                                    const int* __restrict__ active, int band_mod) {
  __shared__ double2 cs[TR][TM];
  __shared__ double2 ps[TM][AS];
  const ProjTile t = a.tiles[blockIdx.x];
  const int g0 = blockIdx.y * AS;
  const int nocc = a.nocc[t.k];
  const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
  const int tr = threadIdx.x >> 4, tg = threadIdx.x & 15;
  double2 acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j] = make_double2(0.0, 0.0);

  for (int mb = 0; mb < nocc; mb += TM) {
    const int mlen = min(TM, nocc - mb);
    for (int e = threadIdx.x; e < TR * TM; e += 128) {
      const int r = e / TM, m = e - r * TM;
      cs[r][m] = (r < t.nrows && m < mlen) ? C[(size_t)(t.row0 + r) * a.ldc + mb + m]
                                           : make_double2(0.0, 0.0);
    }
    for (int e = threadIdx.x; e < TM * AS; e += 128) {
      const int m = e / AS, c = e - m * AS;
      const int g = g0 + c;
      ps[m][c] = (m < mlen && g < a.nbp) ? phi[(size_t)(mb + m) * a.nbp + g]
                                         : make_double2(0.0, 0.0);
    }
    __syncthreads();
#pragma unroll 4
    for (int m = 0; m < TM; ++m) {
      double2 cv[4], pv[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) cv[i] = cs[tr + 8 * i][m];
#pragma unroll
      for (int j = 0; j < 4; ++j) pv[j] = ps[m][tg + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j].x = fma(pv[j].x, cv[i].x, acc[i][j].x);
          acc[i][j].x = fma(-pv[j].y, cv[i].y, acc[i][j].x);
          acc[i][j].y = fma(pv[j].x, cv[i].y, acc[i][j].y);
          acc[i][j].y = fma(pv[j].y, cv[i].x, acc[i][j].y);
        }
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int r = tr + 8 * i;
    if (r >= t.nrows) continue;
    const int row = t.row0 + r;
    if (active && !active[row % band_mod]) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int g = g0 + tg + 16 * j;
      if (g >= a.nbp) continue;
      const size_t idx = (size_t)row * a.nbp + g;
      double2 x = (ca != 0.0) ? Xin[idx] : make_double2(0.0, 0.0);
      Y[idx] = make_double2(ca * x.x + cb * acc[i][j].x, ca * x.y + cb * acc[i][j].y);
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
  pl.mtiles = (maxocc + TM - 1) / TM;
  const int ntiles = (int)pl.tiles.size();
  int want = (2 * kSM + ntiles * pl.mtiles - 1) / std::max(1, ntiles * pl.mtiles);
  int maxsplit = std::max(1, nbp / 64);
  pl.nsplit = std::min(std::max(1, want), maxsplit);
  int len = (nbp + pl.nsplit - 1) / pl.nsplit;
  len = ((len + TS - 1) / TS) * TS;
  pl.split_len = len;
  pl.nsplit = (nbp + len - 1) / len;
  PWB_TRY(pl.dtiles.ensure(pl.tiles.size() * sizeof(ProjTile)));
  if (!pl.tiles.empty())
    PWB_CUDA(cudaMemcpy(pl.dtiles.ptr, pl.tiles.data(), pl.tiles.size() * sizeof(ProjTile),
                        cudaMemcpyHostToDevice));
  return PWB_OK;
}

int proj_coeffs(const ProjPlan& pl, ProjArgs a, const double2* X, double2* part, double2* C,
                cudaStream_t st) {
  if (pl.tiles.empty()) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  dim3 grid((unsigned)pl.tiles.size(), pl.mtiles, pl.nsplit);
  double2* target = (pl.nsplit == 1) ? C : part;
  k_proj_partial<<<grid, 64, 0, st>>>(a, X, pl.split_len, target);
  PWB_LAUNCH_CHECK();
  if (pl.nsplit > 1) {
    const size_t n = (size_t)pl.nrows * a.ldc;
    k_proj_reduce<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(pl.nsplit, n, part, C);
    PWB_LAUNCH_CHECK();
  }
  return PWB_OK;
}

int proj_apply(const ProjPlan& pl, ProjArgs a, const double2* C, const double2* Xin, double2* Y,
               double ca, double cb, const int* active, int band_mod, cudaStream_t st) {
  if (pl.tiles.empty()) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  dim3 grid((unsigned)pl.tiles.size(), (a.nbp + AS - 1) / AS);
  k_proj_apply<<<grid, 128, 0, st>>>(a, C, Xin, Y, ca, cb, active, band_mod > 0 ? band_mod : 1);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

}  // namespace pwb
