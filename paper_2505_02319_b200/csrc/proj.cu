// Occupied-subspace projector Q = 1 - Phi Phi^H as two complex-FP64 GEMMs on
// the FP64 tensor pipe (DMMA: mma.sync.m8n8k4.f64), reference
// sternheimer.py:28-30 and response.py:129,138.
//
//   coef :  C[row][m] = sum_g conj(Phi_k[m][g]) X[row][g]
//           split-K over the sphere; warps of a CTA reduce in smem, splits are
//           reduced in FIXED split order by the last CTA to finish a tile
//           (threadfence + arrival counter): bitwise reproducible, one launch.
//   apply:  Y[row][g] = a X[row][g] + b sum_m Phi_k[m][g] C[row][m]
//
// Both kernels are persistent over a work-item list ((tile, m block, split)
// and (tile, g chunk)) with the grid sized to the SMs, and the number of
// splits is chosen on the device from the live tile count: with active-row
// compaction the tile count shrinks every CG iteration, and a fixed grid of
// mostly-exiting CTAs (or too few splits) was measured to dominate the tail.
//
// Complex products are four real DMMAs (re.re, im.im, re.im, im.re).  Rows of
// X are grouped in tiles of <= 16 rows sharing one k block; with active-row
// compaction the tile rows index X through a row list.
// Measured on B200: DMMA 37.1 TFLOP/s, DFMA 34.0 TFLOP/s (tools/fp64_peak.cu).
#include <cstring>

#include "proj.cuh"

namespace pwb {

constexpr int TR = kProjTileRows;   // rows per tile (2 DMMA n-fragments)
constexpr int CM = 32;   // m per coef block (4 DMMA m-fragments)
constexpr int CW = 8;    // warps per coef CTA
constexpr int AW = 8;    // warps per apply CTA
constexpr int AG = AW * 32;  // g per apply work item (32 per warp)
constexpr int kCoefCtas = 2 * kSM;
constexpr int kApplyCtas = 2 * kSM;

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

// live split count for `units` (tile x m block) work units
__device__ __forceinline__ int live_nsplit(int units, int nsplit_max) {
  int s = (kCoefCtas + units - 1) / max(units, 1);
  return max(1, min(s, nsplit_max));
}

__global__ void __launch_bounds__(CW * 32) k_proj_coef(ProjArgs a, const double2* __restrict__ X,
                                                       int nt_host, int tile_cap, int mtiles,
                                                       int nsplit_max, double2* __restrict__ part,
                                                       double2* __restrict__ C,
                                                       unsigned* __restrict__ counters) {
  __shared__ double2 red[CW / 2][CM][TR];
  __shared__ bool last;
  const int ntiles = a.ntiles ? *a.ntiles : nt_host;
  const int units = ntiles * mtiles;
  const int nsplit = live_nsplit(units, nsplit_max);
  int split_len = (a.nbp + nsplit - 1) / nsplit;
  split_len = ((split_len + 4 * CW - 1) / (4 * CW)) * (4 * CW);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  const size_t stride = (size_t)tile_cap * mtiles * (CM * TR);   // per split
  for (int item = blockIdx.x; item < units * nsplit; item += gridDim.x) {
    const int split = item % nsplit;
    const int unit = item / nsplit;
    const int mblk = unit % mtiles, tile = unit / mtiles;
    const ProjTile t = a.tiles[tile];
    const int m0 = mblk * CM;
    const int nocc = a.nocc[t.k];
    if (m0 >= nocc) continue;   // uniform over the CTA
    const int g0 = split * split_len;
    const int g1 = min(a.nbp, g0 + split_len);
    const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
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
      xrw[nb] = X + (size_t)(xok[nb] ? (a.rows ? a.rows[t.row0 + r] : t.row0 + r) : 0) * a.nbp;
    }
    double cr[4][2][2], ci[4][2][2];
#pragma unroll
    for (int ma = 0; ma < 4; ++ma)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        cr[ma][nb][0] = cr[ma][nb][1] = 0.0;
        ci[ma][nb][0] = ci[ma][nb][1] = 0.0;
      }
    // batched prefetch: the fragments of NP k-steps are loaded before any is used
    constexpr int NP = 4;
    for (int gb = g0 + 4 * w; gb < g1; gb += 4 * CW * NP) {
      double2 av[NP][4], bv[NP][2];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int gg = gb + 4 * CW * u + c4;
        const bool gok = gg < g1;
#pragma unroll
        for (int ma = 0; ma < 4; ++ma)
          av[u][ma] = (gok && pok[ma]) ? __ldg(&prow[ma][gg]) : make_double2(0.0, 0.0);
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
          bv[u][nb] = (gok && xok[nb]) ? xrw[nb][gg] : make_double2(0.0, 0.0);
      }
      // conj(phi) * x : re = pr xr + pi xi ; im = pr xi - pi xr (part-major issue)
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int ma = 0; ma < 4; ++ma)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            dmma(cr[ma][nb][0], cr[ma][nb][1], av[u][ma].x, bv[u][nb].x);
            dmma(ci[ma][nb][0], ci[ma][nb][1], av[u][ma].x, bv[u][nb].y);
          }
#pragma unroll
        for (int ma = 0; ma < 4; ++ma)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            dmma(cr[ma][nb][0], cr[ma][nb][1], av[u][ma].y, bv[u][nb].y);
            dmma(ci[ma][nb][0], ci[ma][nb][1], -av[u][ma].y, bv[u][nb].x);
          }
      }
    }
    // fixed-order warp reduction in two halves: warp w (< CW/2) adds w + CW/2
    if (w >= CW / 2) {
#pragma unroll
      for (int ma = 0; ma < 4; ++ma)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            red[w - CW / 2][8 * ma + r4][8 * nb + 2 * c4 + h] =
                make_double2(cr[ma][nb][h], ci[ma][nb][h]);
    }
    __syncthreads();
    if (w < CW / 2) {
#pragma unroll
      for (int ma = 0; ma < 4; ++ma)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double2& slot = red[w][8 * ma + r4][8 * nb + 2 * c4 + h];
            slot = make_double2(cr[ma][nb][h] + slot.x, ci[ma][nb][h] + slot.y);
          }
    }
    __syncthreads();
    const size_t tile_id = (size_t)tile * mtiles + mblk;
    double2* mypart = part + (size_t)split * stride + tile_id * (CM * TR);
    for (int i = threadIdx.x; i < CM * TR; i += CW * 32) {
      const int m = i / TR, r = i - m * TR;
      double2 s = red[0][m][r];
#pragma unroll
      for (int q = 1; q < CW / 2; ++q) s = cadd(s, red[q][m][r]);
      if (nsplit == 1) {
        if (r < t.nrows && m0 + m < nocc) C[(size_t)(t.row0 + r) * a.ldc + m0 + m] = s;
      } else {
        mypart[i] = s;
      }
    }
    if (nsplit > 1) {
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&counters[tile_id], 1u);
        last = (prev == (unsigned)nsplit - 1);
      }
      __syncthreads();
      if (last) {
        __threadfence();
        const double2* p0 = part + tile_id * (CM * TR);
        for (int i = threadIdx.x; i < CM * TR; i += CW * 32) {
          const int m = i / TR, r = i - m * TR;
          double2 s = __ldcg(&p0[i]);
          int q = 1;
          // loads issued 8 at a time (serialised on L2 latency otherwise), summed in order
          for (; q + 8 <= nsplit; q += 8) {
            double2 v[8];
#pragma unroll
            for (int u = 0; u < 8; ++u) v[u] = __ldcg(&p0[(size_t)(q + u) * stride + i]);
#pragma unroll
            for (int u = 0; u < 8; ++u) s = cadd(s, v[u]);
          }
          for (; q < nsplit; ++q) s = cadd(s, __ldcg(&p0[(size_t)q * stride + i]));
          if (r < t.nrows && m0 + m < nocc) C[(size_t)(t.row0 + r) * a.ldc + m0 + m] = s;
        }
        if (threadIdx.x == 0) counters[tile_id] = 0u;
      }
    }
    __syncthreads();   // red / last reused by the next item
  }
}

// work item = (tile, chunk of AG g); warp w covers g0 + 32 w .. + 32
__global__ void __launch_bounds__(AW * 32) k_proj_apply(ProjArgs a, const double2* __restrict__ C,
                                                        const double2* __restrict__ Xin,
                                                        double2* __restrict__ Y, double ca,
                                                        double cb, const int* __restrict__ active,
                                                        int band_mod, int nt_host) {
  const int ntiles = a.ntiles ? *a.ntiles : nt_host;
  const int nchunk = (a.nbp + AG - 1) / AG;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  for (int item = blockIdx.x; item < ntiles * nchunk; item += gridDim.x) {
    const int tile = item / nchunk, chunk = item - tile * nchunk;
    const ProjTile t = a.tiles[tile];
    const int nocc = a.nocc[t.k];
    const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
    const int gw = chunk * AG + 32 * w;
    if (gw >= a.nbp) continue;   // per warp: no block-level sync below
    double dr[2][4][2], di[2][4][2];
#pragma unroll
    for (int jb = 0; jb < 2; ++jb)
#pragma unroll
      for (int gb = 0; gb < 4; ++gb) {
        dr[jb][gb][0] = dr[jb][gb][1] = 0.0;
        di[jb][gb][0] = di[jb][gb][1] = 0.0;
      }
    // batched prefetch of NP m-steps (all of nocc = 32 in one batch)
    constexpr int NP = 8;
    for (int mb = 0; mb < nocc; mb += 4 * NP) {
      double2 av[NP][2], bv[NP][4];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int mm = mb + 4 * u + c4;
        const bool mok = mm < nocc;
#pragma unroll
        for (int jb = 0; jb < 2; ++jb) {
          const int r = 8 * jb + r4;   // A[j = r4][k = c4] = C[row j][m + c4]
          av[u][jb] = (mok && r < t.nrows) ? C[(size_t)(t.row0 + r) * a.ldc + mm]
                                           : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int gb = 0; gb < 4; ++gb) {
          const int g = gw + 8 * gb + r4;   // B[k = c4][n = r4] = Phi[m + c4][g]
          bv[u][gb] = (mok && g < a.nbp) ? __ldg(&phi[(size_t)mm * a.nbp + g])
                                         : make_double2(0.0, 0.0);
        }
      }
      // C * Phi : re = cr pr - ci pi ; im = cr pi + ci pr (part-major issue order)
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int jb = 0; jb < 2; ++jb)
#pragma unroll
          for (int gb = 0; gb < 4; ++gb) {
            dmma(dr[jb][gb][0], dr[jb][gb][1], av[u][jb].x, bv[u][gb].x);
            dmma(di[jb][gb][0], di[jb][gb][1], av[u][jb].x, bv[u][gb].y);
          }
#pragma unroll
        for (int jb = 0; jb < 2; ++jb)
#pragma unroll
          for (int gb = 0; gb < 4; ++gb) {
            dmma(dr[jb][gb][0], dr[jb][gb][1], -av[u][jb].y, bv[u][gb].y);
            dmma(di[jb][gb][0], di[jb][gb][1], av[u][jb].y, bv[u][gb].x);
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
}

int proj_plan(ProjPlan& pl, const std::vector<int>& row_k, const std::vector<int>& nocc,
              int nbp, cudaStream_t st, bool async) {
  pl.tiles.clear();
  pl.max_tiles = 0;
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
  pl.mtiles = std::max(1, (maxocc + CM - 1) / CM);
  const int ntiles = (int)pl.tiles.size();
  pl.nsplit = std::max(1, std::min(kCoefCtas, nbp / (16 * CW)));   // upper bound
  PWB_TRY(pl.dtiles.ensure(std::max<size_t>(1, pl.tiles.size()) * sizeof(ProjTile)));
  if (!pl.tiles.empty()) {
    if (async) {
      if (pl.h_cap < pl.tiles.size()) {
        if (pl.h_stage) cudaFreeHost(pl.h_stage);
        pl.h_cap = std::max<size_t>(64, 2 * pl.tiles.size());
        PWB_CUDA(cudaMallocHost(&pl.h_stage, pl.h_cap * sizeof(ProjTile)));
      }
      memcpy(pl.h_stage, pl.tiles.data(), pl.tiles.size() * sizeof(ProjTile));
      PWB_CUDA(cudaMemcpyAsync(pl.dtiles.ptr, pl.h_stage, pl.tiles.size() * sizeof(ProjTile),
                               cudaMemcpyHostToDevice, st));
    } else {
      PWB_CUDA(cudaMemcpy(pl.dtiles.ptr, pl.tiles.data(), pl.tiles.size() * sizeof(ProjTile),
                          cudaMemcpyHostToDevice));
    }
  }
  const size_t ntm = (size_t)std::max(1, ntiles) * pl.mtiles;
  if (pl.counters.bytes < ntm * sizeof(unsigned) || !pl.counters.ptr) {
    PWB_TRY(pl.counters.ensure(ntm * sizeof(unsigned)));
    PWB_CUDA(cudaMemset(pl.counters.ptr, 0, ntm * sizeof(unsigned)));
  }
  return PWB_OK;
}

size_t proj_part_elems(const ProjPlan& pl) {
  return (size_t)pl.nsplit * std::max(1, plan_tiles(pl)) * pl.mtiles * CM * TR;
}

int proj_plan_device(ProjPlan& pl, int max_tiles, int maxocc, int nbp) {
  pl.tiles.clear();
  pl.max_tiles = max_tiles;
  pl.nrows = max_tiles * TR;
  pl.mtiles = std::max(1, (maxocc + CM - 1) / CM);
  pl.nsplit = std::max(1, std::min(kCoefCtas, nbp / (16 * CW)));   // upper bound
  PWB_TRY(pl.dtiles.ensure(std::max<size_t>(1, max_tiles) * sizeof(ProjTile)));
  const size_t ntm = (size_t)std::max(1, max_tiles) * pl.mtiles;
  PWB_TRY(pl.counters.ensure(ntm * sizeof(unsigned)));
  PWB_CUDA(cudaMemset(pl.counters.ptr, 0, ntm * sizeof(unsigned)));
  return PWB_OK;
}

int proj_coeffs(const ProjPlan& pl, ProjArgs a, const double2* X, double2* part, double2* C,
                cudaStream_t st) {
  const int cap = plan_tiles(pl);
  if (cap == 0) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  const long items = (long)cap * pl.mtiles * pl.nsplit;
  const int grid = (int)std::min<long>(items, kCoefCtas);
  k_proj_coef<<<grid, CW * 32, 0, st>>>(a, X, (int)pl.tiles.size(), cap, pl.mtiles, pl.nsplit,
                                        part, C, reinterpret_cast<unsigned*>(pl.counters.ptr));
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int proj_apply(const ProjPlan& pl, ProjArgs a, const double2* C, const double2* Xin, double2* Y,
               double ca, double cb, const int* active, int band_mod, cudaStream_t st) {
  const int cap = plan_tiles(pl);
  if (cap == 0) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  const long items = (long)cap * ((a.nbp + AG - 1) / AG);
  const int grid = (int)std::min<long>(items, kApplyCtas);
  k_proj_apply<<<grid, AW * 32, 0, st>>>(a, C, Xin, Y, ca, cb, active,
                                         band_mod > 0 ? band_mod : 1, (int)pl.tiles.size());
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

// ---------------------------------------------------------------------------
// Fused Q in ONE launch with a thread-block cluster per row tile:
//   CTA c of the cluster owns g in [c L, (c+1) L);
//   phase 1: partial C = Phi^H X over its g range (DMMA), warp-reduced in smem;
//   cluster barrier; every CTA sums the CS partials through DSMEM in rank
//   order (deterministic) -> full C in its own smem; cluster barrier;
//   phase 2: Y = ca X + cb Phi C on its g range with C read from smem.
// No global partial buffer, no atomics, one launch instead of two.
}  // namespace pwb

#include <cooperative_groups.h>

namespace pwb {

constexpr int QW = 8;          // warps per CTA
constexpr int QCS = 8;         // CTAs per cluster (g split)

__global__ void __launch_bounds__(QW * 32) k_proj_q(ProjArgs a, const double2* __restrict__ Xin,
                                                    double2* __restrict__ Y, double ca, double cb,
                                                    const int* __restrict__ active, int band_mod,
                                                    int glen) {
  namespace cgp = cooperative_groups;
  cgp::cluster_group cluster = cgp::this_cluster();
  extern __shared__ double2 qsm[];
  const int tile = blockIdx.x / QCS;
  const int crank = (int)cluster.block_rank();
  if (a.ntiles && tile >= *a.ntiles) return;   // whole cluster exits together
  const ProjTile t = a.tiles[tile];
  const int nocc = a.nocc[t.k];
  const int ldm = ((a.ldc + 31) / 32) * 32;    // m capacity of the smem C blocks
  double2* red = qsm;                          // [QW/2][CM][TR]
  double2* cpart = red + (QW / 2) * CM * TR;   // [ldm][TR] this CTA's partial
  double2* cfull = cpart + ldm * TR;           // [ldm][TR] cluster sum
  const double2* phi = a.phi + (size_t)a.off[t.k] * a.nbp;
  const int g0 = crank * glen;
  const int g1 = min(a.nbp, g0 + glen);
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;

  const double2* xrw[2];
  bool xok[2];
#pragma unroll
  for (int nb = 0; nb < 2; ++nb) {
    const int r = 8 * nb + r4;
    xok[nb] = r < t.nrows;
    xrw[nb] = Xin + (size_t)(xok[nb] ? (a.rows ? a.rows[t.row0 + r] : t.row0 + r) : 0) * a.nbp;
  }
  // ---- phase 1: partial C over this CTA's g range, 32 m at a time
  for (int m0 = 0; m0 < nocc; m0 += CM) {
    const double2* prow[4];
    bool pok[4];
#pragma unroll
    for (int ma = 0; ma < 4; ++ma) {
      const int m = m0 + 8 * ma + r4;
      pok[ma] = m < nocc;
      prow[ma] = phi + (size_t)(pok[ma] ? m : 0) * a.nbp;
    }
    double cr[4][2][2], ci[4][2][2];
#pragma unroll
    for (int ma = 0; ma < 4; ++ma)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        cr[ma][nb][0] = cr[ma][nb][1] = 0.0;
        ci[ma][nb][0] = ci[ma][nb][1] = 0.0;
      }
    constexpr int NP = 4;
    for (int gb = g0 + 4 * w; gb < g1; gb += 4 * QW * NP) {
      double2 av[NP][4], bv[NP][2];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int gg = gb + 4 * QW * u + c4;
        const bool gok = gg < g1;
#pragma unroll
        for (int ma = 0; ma < 4; ++ma)
          av[u][ma] = (gok && pok[ma]) ? __ldg(&prow[ma][gg]) : make_double2(0.0, 0.0);
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
          bv[u][nb] = (gok && xok[nb]) ? xrw[nb][gg] : make_double2(0.0, 0.0);
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int ma = 0; ma < 4; ++ma)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            dmma(cr[ma][nb][0], cr[ma][nb][1], av[u][ma].x, bv[u][nb].x);
            dmma(ci[ma][nb][0], ci[ma][nb][1], av[u][ma].x, bv[u][nb].y);
          }
#pragma unroll
        for (int ma = 0; ma < 4; ++ma)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb) {
            dmma(cr[ma][nb][0], cr[ma][nb][1], av[u][ma].y, bv[u][nb].y);
            dmma(ci[ma][nb][0], ci[ma][nb][1], -av[u][ma].y, bv[u][nb].x);
          }
      }
    }
    // fixed-order warp reduction -> cpart[m0 + m][r]
    if (w >= QW / 2) {
#pragma unroll
      for (int ma = 0; ma < 4; ++ma)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h)
            red[((w - QW / 2) * CM + 8 * ma + r4) * TR + 8 * nb + 2 * c4 + h] =
                make_double2(cr[ma][nb][h], ci[ma][nb][h]);
    }
    __syncthreads();
    if (w < QW / 2) {
#pragma unroll
      for (int ma = 0; ma < 4; ++ma)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb)
#pragma unroll
          for (int h = 0; h < 2; ++h) {
            double2& slot = red[(w * CM + 8 * ma + r4) * TR + 8 * nb + 2 * c4 + h];
            slot = make_double2(cr[ma][nb][h] + slot.x, ci[ma][nb][h] + slot.y);
          }
    }
    __syncthreads();
    for (int i = threadIdx.x; i < CM * TR; i += QW * 32) {
      double2 s = red[i];
#pragma unroll
      for (int q = 1; q < QW / 2; ++q) s = cadd(s, red[q * CM * TR + i]);
      cpart[m0 * TR + i] = s;
    }
    __syncthreads();
  }
  // ---- cluster reduction through DSMEM, rank order
  cluster.sync();
  for (int i = threadIdx.x; i < nocc * TR; i += QW * 32) {
    double2 s = make_double2(0.0, 0.0);
    for (int c = 0; c < QCS; ++c) {
      const double2* rp = cluster.map_shared_rank(cpart, c);
      s = cadd(s, rp[i]);
    }
    cfull[i] = s;
  }
  cluster.sync();   // no CTA may leave while its cpart is still being read
  // ---- phase 2: Y = ca X + cb Phi C on this CTA's g range
  for (int gw = g0 + 32 * w; gw < g1; gw += 32 * QW) {
    double dr[2][4][2], di[2][4][2];
#pragma unroll
    for (int jb = 0; jb < 2; ++jb)
#pragma unroll
      for (int gb = 0; gb < 4; ++gb) {
        dr[jb][gb][0] = dr[jb][gb][1] = 0.0;
        di[jb][gb][0] = di[jb][gb][1] = 0.0;
      }
    constexpr int NP = 8;
    for (int mb = 0; mb < nocc; mb += 4 * NP) {
      double2 av[NP][2], bv[NP][4];
#pragma unroll
      for (int u = 0; u < NP; ++u) {
        const int mm = mb + 4 * u + c4;
        const bool mok = mm < nocc;
#pragma unroll
        for (int jb = 0; jb < 2; ++jb)   // A[j = r4][k = c4] = C[row j][m]
          av[u][jb] = mok ? cfull[mm * TR + 8 * jb + r4] : make_double2(0.0, 0.0);
#pragma unroll
        for (int gb = 0; gb < 4; ++gb) {
          const int g = gw + 8 * gb + r4;   // B[k = c4][n = r4] = Phi[m][g]
          bv[u][gb] = (mok && g < g1) ? __ldg(&phi[(size_t)mm * a.nbp + g])
                                      : make_double2(0.0, 0.0);
        }
      }
#pragma unroll
      for (int u = 0; u < NP; ++u) {
#pragma unroll
        for (int jb = 0; jb < 2; ++jb)
#pragma unroll
          for (int gb = 0; gb < 4; ++gb) {
            dmma(dr[jb][gb][0], dr[jb][gb][1], av[u][jb].x, bv[u][gb].x);
            dmma(di[jb][gb][0], di[jb][gb][1], av[u][jb].x, bv[u][gb].y);
          }
#pragma unroll
        for (int jb = 0; jb < 2; ++jb)
#pragma unroll
          for (int gb = 0; gb < 4; ++gb) {
            dmma(dr[jb][gb][0], dr[jb][gb][1], -av[u][jb].y, bv[u][gb].y);
            dmma(di[jb][gb][0], di[jb][gb][1], av[u][jb].y, bv[u][gb].x);
          }
      }
    }
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
          if (g >= g1) continue;
          const size_t idx = (size_t)row * a.nbp + g;
          const double2 x = (ca != 0.0) ? Xin[idx] : make_double2(0.0, 0.0);
          Y[idx] = make_double2(ca * x.x + cb * dr[jb][gb][h], ca * x.y + cb * di[jb][gb][h]);
        }
    }
  }
}

size_t proj_q_smem(int ldc) {
  const int ldm = ((ldc + 31) / 32) * 32;
  return ((size_t)(QW / 2) * CM * TR + 2 * (size_t)ldm * TR) * sizeof(double2);
}

int proj_q(const ProjPlan& pl, ProjArgs a, const double2* Xin, double2* Y, double ca, double cb,
           const int* active, int band_mod, cudaStream_t st) {
  const int nt = plan_tiles(pl);
  if (nt == 0) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  int glen = (a.nbp + QCS - 1) / QCS;
  glen = ((glen + 31) / 32) * 32;
  const size_t smem = proj_q_smem(a.ldc);
  static bool configured = false;
  static size_t configured_smem = 0;
  if (!configured || smem > configured_smem) {
    PWB_CUDA(cudaFuncSetAttribute(k_proj_q, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  (int)std::max<size_t>(smem, 48 * 1024)));
    configured = true;
    configured_smem = std::max<size_t>(smem, 48 * 1024);
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)(nt * QCS), 1, 1);
  cfg.blockDim = dim3(QW * 32, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = QCS;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  PWB_CUDA(cudaLaunchKernelEx(&cfg, k_proj_q, a, Xin, Y, ca, cb, active,
                              band_mod > 0 ? band_mod : 1, glen));
  count_launch();
  return PWB_OK;
}

}  // namespace pwb
