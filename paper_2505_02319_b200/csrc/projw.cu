// Wide-tile projector: Q X = X - Phi (Phi^H X) with one tile = up to 72 rows
// of ONE k block against ALL its orbitals (<= 72), reference
// sternheimer.py:28-30.  This is the shape of a Sternheimer batch at full
// width (every occupied band of a k point iterates: rows_k = N_occ,k), where
// the 16-row tiles of proj.cu re-stream Phi_k once per 16 rows and the X rows
// once per 40-orbital block.  Here both operands cross L2 -> SM exactly once
// per tile:
//
//   coef :  C[row][m] = sum_g conj(Phi_k[m][g]) X[row][g]
//           stream-K over (tile, 32-coefficient chunk) units: every CTA of the
//           persistent grid takes an equal contiguous run of units; a tile cut
//           between CTAs leaves per-CTA partial C blocks that the last CTA to
//           arrive sums in fixed CTA order (bitwise reproducible, one launch).
//   apply:  Y[row][g] = a X[row][g] + b sum_m Phi_k[m][g] C[row][m]
//           contiguous runs of (tile, chunk) units per CTA; the tile's C block
//           stays in smem across its chunks.
//
// Operands arrive by TMA bulk copies (one copy for the chunk's Phi block from
// the 32-wide chunk-major copy, one 512 B copy per gathered X row) into an
// smem ring with full/empty mbarriers; warp 0 refills a stage once every warp
// has released it (no separate producer warp).  Twelve compute warps -- three
// per SM sub-partition, so the four DMMA pipes are loaded evenly (nine warps
// cap the busiest sub-partition at 3 of 4 warps' worth: 75%) -- form a 4 x 3
// grid over the output fragments (8 x 8 DMMA tiles, mma.sync.m8n8k4.f64 ->
// DMMA.8x8x4), so a warp reuses each loaded A fragment across its n
// fragments and vice versa; complex products use three real DMMAs (Gauss),
// as in proj.cu.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cstring>
#include <mutex>

#include "proj.cuh"
#include "tma.cuh"

namespace pwb {

constexpr int WR = kProjWideRows;    // rows per wide tile (9 n fragments)
constexpr int WMO = kProjWideOcc;    // orbitals per k block (9 m fragments)
#ifndef PWB_WKC
#define PWB_WKC 32   // coef chunk (coefficients): 2 stages of 83 KB (16 x 4 stages measured 28% slower)
#endif
constexpr int KWC = PWB_WKC;             // coef: coefficients per chunk
constexpr int RSWC = KWC + 4;            // coef smem / chunk-major row stride (double2): the
                                         // A/B fragment loads (8 rows x 4 columns) need 4 mod 8
constexpr int KWA = kProjWideChunk;      // apply: coefficients per chunk (32)
constexpr int RSWA = KWA + 6;            // apply row stride: the B loads (4 rows x 8
                                         // columns) need 2 or 6 mod 8 (38: conflict-free)
constexpr int NWW = 12;                  // compute warps (3 per SM sub-partition)
constexpr int WST = KWC == 16 ? 4 : 2;   // coef pipeline stages
constexpr int WSA = 3;                   // apply pipeline stages
constexpr int kWCoefStage = (WR + WMO) * RSWC;   // double2: X rows, then the Phi block
constexpr int kWApplyStage = WMO * RSWA;         // double2: the Phi block
constexpr int kWCs = WMO + 4;                    // C tile smem stride (4 mod 8: conflict-free)
constexpr size_t kWCoefSmem = (size_t)WST * kWCoefStage * 16 + 64;
constexpr size_t kWApplySmem = (size_t)WSA * kWApplyStage * 16 + (size_t)WR * kWCs * 16 + 64;
static_assert(kWCoefSmem <= 232448 && kWApplySmem <= 232448, "wide projector smem");
static_assert(RSWC % 8 == 4 && (RSWA % 8 == 2 || RSWA % 8 == 6), "bank-conflict-free strides");
constexpr int kWThreads = NWW * 32;

__device__ __forceinline__ void wdmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}


__device__ __forceinline__ int wxrow(const ProjArgs& a, const ProjTile& t, int r) {
  return a.rows ? a.rows[t.row0 + r] : t.row0 + r;
}

// chunk-major Phi blocks: orbitals 0 .. nocc-1 of chunk c of block k, in the coef
// (KWC-wide, stride RSWC) and apply (KWA-wide, stride RSWA) copies
__device__ __forceinline__ const double2* phiw_at(const ProjArgs& a, int k, int nocc, int c) {
  return a.phiw + a.phiw_off[k] + (size_t)c * nocc * RSWC;
}
__device__ __forceinline__ const double2* phiwa_at(const ProjArgs& a, int k, int nocc, int c) {
  return a.phiwa + a.phiwa_off[k] + (size_t)c * nocc * RSWA;
}

// balanced split of n fragments over `parts` warps: [lo, hi) of part p
__device__ __forceinline__ void splitn(int n, int p, int parts, int& lo, int& hi) {
  lo = (p * n) / parts;
  hi = ((p + 1) * n) / parts;
}

// TMA tensor maps of X, one per box height 8, 16, ..., 72 rows: a tile is loaded
// with the box of its own height.  (One 72-row box for every tile made the TMA unit
// move 41 KB of X per stage whatever the tile held -- 72 rows of 576 B each; at
// 24-48 rows per tile that copy, not the DMMAs, set the stage time:
// tools/qmid.py, 48 rows per k cost what 66 did.)
struct XMaps {
  CUtensorMap m[WR / 8];
};

// One 32-coefficient chunk of a warp's CM x CN output fragments (coef kernel).  The
// fragment counts are template parameters: with runtime bounds and `break`s in the
// unrolled loops nvcc kept the branch for the first fragment but ran the second and
// third speculatively (DMMAs have no side effects), so a 48-row tile (2 n fragments
// per warp) executed the DMMAs of a 72-row one (ncu: 31.1 M DMMA at 48 and at 66 rows).
template <int CM, int CN>
__device__ __forceinline__ void coef_chunk(const double2* __restrict__ xb,
                                           const double2* __restrict__ pb, double (&t1)[3][3][2],
                                           double (&t2)[3][3][2], double (&t3)[3][3][2]) {
#pragma unroll 2
  for (int kk = 0; kk < KWC / 4; ++kk) {
    double2 bv[CN];
    double bs[CN];
#pragma unroll
    for (int j = 0; j < CN; ++j) {
      bv[j] = xb[8 * j * RSWC + 4 * kk];
      bs[j] = bv[j].x + bv[j].y;
    }
    // conj(phi) x: re = pr xr + pi xi, im = pr xi - pi xr (3 real products)
#pragma unroll
    for (int i = 0; i < CM; ++i) {
      const double2 av = pb[8 * i * RSWC + 4 * kk];
      const double ad = av.x - av.y;
#pragma unroll
      for (int j = 0; j < CN; ++j) {
        wdmma(t1[i][j][0], t1[i][j][1], av.x, bv[j].x);
        wdmma(t2[i][j][0], t2[i][j][1], av.y, bv[j].y);
        wdmma(t3[i][j][0], t3[i][j][1], ad, bs[j]);
      }
    }
  }
}

// One 32-coefficient chunk of a warp's CR row fragments x one g fragment (apply
// kernel), software-pipelined over the orbital steps: the next step's fragments are
// loaded from smem before this step's DMMAs issue (3 warps per sub-partition leave
// too little parallelism to hide the LDS latency otherwise).
template <int CR>
__device__ __forceinline__ void apply_chunk(const double2* __restrict__ ps,
                                            const double2* __restrict__ ca, int nm, int c4,
                                            double (&t1)[3][2], double (&t2)[3][2],
                                            double (&t3)[3][2]) {
  auto ldb = [&](int ms) {   // B[k = c4][n = r4] = Phi[m][g]
    const int m = ms + c4;
    return m < nm ? ps[m * RSWA] : make_double2(0.0, 0.0);
  };
  auto lda = [&](int ms, int i) {   // A[j = r4][k = c4] = C[row][m]; padding exactly zero
    const int m = ms + c4;
    return m < nm ? ca[8 * i * kWCs + m] : make_double2(0.0, 0.0);
  };
  double2 bv = ldb(0), av[CR];
#pragma unroll
  for (int i = 0; i < CR; ++i) av[i] = lda(0, i);
  for (int ms = 0; ms < nm; ms += 4) {
    const double2 bn = ldb(ms + 4);
    double2 an[CR];
#pragma unroll
    for (int i = 0; i < CR; ++i) an[i] = lda(ms + 4, i);
    const double bs = bv.x + bv.y;
    // c phi: re = cr pr - ci pi, im = cr pi + ci pr (3 real products)
#pragma unroll
    for (int i = 0; i < CR; ++i) {
      wdmma(t1[i][0], t1[i][1], av[i].x, bv.x);
      wdmma(t2[i][0], t2[i][1], av[i].y, bv.y);
      wdmma(t3[i][0], t3[i][1], av[i].x + av[i].y, bs);
    }
    bv = bn;
#pragma unroll
    for (int i = 0; i < CR; ++i) av[i] = an[i];
  }
}

struct WRange {
  int u0, u1, nch;   // this CTA's units [u0, u1); chunks per tile
};

__device__ __forceinline__ WRange wrange(const ProjArgs& a, int nt_host, int kw) {
  const int ntiles = a.ntiles ? *a.ntiles : nt_host;
  WRange r;
  r.nch = a.nbp / kw;
  const long long units = (long long)ntiles * r.nch;
  const long long per = (units + gridDim.x - 1) / gridDim.x;
  r.u0 = (int)min(units, per * blockIdx.x);
  r.u1 = (int)min(units, per * (blockIdx.x + 1));
  return r;
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWThreads, 1)
    k_projw_coef(ProjArgs a, const double2* __restrict__ X, int nt_host,
                 double2* __restrict__ part, double2* __restrict__ C,
                 unsigned* __restrict__ counters, const __grid_constant__ XMaps xmaps,
                 int use_map) {
  pdl_wait();
  extern __shared__ __align__(128) double2 sm[];
  uint64_t* full = reinterpret_cast<uint64_t*>(sm + WST * kWCoefStage);
  uint64_t* empty = full + WST;
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WRange R = wrange(a, nt_host, KWC);
  if (threadIdx.x == 0) {
    for (int s = 0; s < WST; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (R.u0 >= R.u1) return;
  // warp 0 fills stage s with unit u: one Phi block copy, and the tile's X rows as
  // ONE 2-D tensor copy (box 72 rows x RSWC complex, the smem row stride) when they
  // are consecutive rows of X, else one bulk copy per row (compacted CG tail).
  // The tile's metadata (tile entry, N_occ, row indices: a chain of dependent global
  // loads) is fetched once per TILE, not per unit: warp 0 is a compute warp too, and
  // ~1 us of load latency per fill sat on every stage's critical path.
  int f_tile = -1, f_nocc = 0, f_x0 = 0, f_rows[3] = {0, 0, 0};
  ProjTile f_t{0, 0, 0};
  bool f_box = false;
  auto fill = [&](int u, int s) {
    const int tile = u / R.nch, c = u - tile * R.nch;
    if (tile != f_tile) {
      f_tile = tile;
      f_t = a.tiles[tile];
      f_nocc = a.nocc[f_t.k];
      f_x0 = wxrow(a, f_t, 0);
      f_box = use_map && wxrow(a, f_t, f_t.nrows - 1) - f_x0 == f_t.nrows - 1;
      if (!f_box)
#pragma unroll
        for (int q = 0; q < 3; ++q)
          f_rows[q] = lane + 32 * q < f_t.nrows ? wxrow(a, f_t, lane + 32 * q) : 0;
    }
    double2* buf = sm + s * kWCoefStage;
    if (lane == 0) {
      const uint32_t pb = (uint32_t)f_nocc * RSWC * 16;
      const int hb = (f_t.nrows + 7) >> 3;   // box height in fragments: the map of that height
      mbar_expect_tx(&full[s], pb + (f_box ? (uint32_t)(8 * hb) * RSWC * 16
                                           : (uint32_t)f_t.nrows * KWC * 16));
      bulk_g2s(buf + WR * RSWC, phiw_at(a, f_t.k, f_nocc, c), pb, &full[s]);
      if (f_box)
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
            " [%0], [%1, {%2, %3}], [%4];\n" ::"r"(su32(buf)),
            "l"(reinterpret_cast<uint64_t>(&xmaps.m[hb - 1])), "r"(2 * KWC * c), "r"(f_x0),
            "r"(su32(&full[s]))
            : "memory");
    }
    if (f_box) return;
    __syncwarp();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      const int r = lane + 32 * q;
      if (r < f_t.nrows)
        bulk_g2s(buf + r * RSWC, X + (size_t)f_rows[q] * a.nbp + (size_t)c * KWC, KWC * 16,
                 &full[s]);
    }
  };
  if (w == 0)
    for (int q = 0; q < WST && R.u0 + q < R.u1; ++q) fill(R.u0 + q, q);
  const int r4 = lane >> 2, c4 = lane & 3;
  const int wm = w / 3, wn = w - 3 * (w / 3);   // 4 (m) x 3 (n) warp grid
  double t1[3][3][2], t2[3][3][2], t3[3][3][2];
  int seq = 0;
  for (int u = R.u0; u < R.u1;) {
    const int tile = u / R.nch;
    const int uend = min(R.u1, (tile + 1) * R.nch);   // this CTA's run on the tile
    const ProjTile t = a.tiles[tile];
    const int nm = a.nocc[t.k];
    int m_lo, m_hi, n_lo, n_hi;
    splitn((nm + 7) >> 3, wm, 4, m_lo, m_hi);
    splitn((t.nrows + 7) >> 3, wn, 3, n_lo, n_hi);
    const int cm = m_hi - m_lo, cn = n_hi - n_lo;
#pragma unroll
    for (int i = 0; i < 3; ++i)
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        t1[i][j][0] = t1[i][j][1] = 0.0;
        t2[i][j][0] = t2[i][j][1] = 0.0;
        t3[i][j][0] = t3[i][j][1] = 0.0;
      }
    for (; u < uend; ++u, ++seq) {
      const int s = seq % WST;
      mbar_wait(&full[s], (seq / WST) & 1);
      const double2* xs = sm + s * kWCoefStage;
      const double2* ps = xs + WR * RSWC;
      {
        const double2* xb = xs + (8 * n_lo + r4) * RSWC + c4;
        const double2* pb = ps + (8 * m_lo + r4) * RSWC + c4;
        switch (4 * cm + cn) {   // warp-uniform; one straight-line body per fragment count
          case 4 * 1 + 1: coef_chunk<1, 1>(xb, pb, t1, t2, t3); break;
          case 4 * 1 + 2: coef_chunk<1, 2>(xb, pb, t1, t2, t3); break;
          case 4 * 1 + 3: coef_chunk<1, 3>(xb, pb, t1, t2, t3); break;
          case 4 * 2 + 1: coef_chunk<2, 1>(xb, pb, t1, t2, t3); break;
          case 4 * 2 + 2: coef_chunk<2, 2>(xb, pb, t1, t2, t3); break;
          case 4 * 2 + 3: coef_chunk<2, 3>(xb, pb, t1, t2, t3); break;
          case 4 * 3 + 1: coef_chunk<3, 1>(xb, pb, t1, t2, t3); break;
          case 4 * 3 + 2: coef_chunk<3, 2>(xb, pb, t1, t2, t3); break;
          case 4 * 3 + 3: coef_chunk<3, 3>(xb, pb, t1, t2, t3); break;
          default: break;   // this warp has no fragment of the tile
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (w == 0 && u + WST < R.u1) {   // refill stage s once every warp released it
        mbar_wait(&empty[s], (seq / WST) & 1);
        fill(u + WST, s);
      }
    }
    // ---- flush the run on `tile`: final C, or a partial + fixed-order reduction
    const int ntiles = a.ntiles ? *a.ntiles : nt_host;
    const long long units = (long long)ntiles * R.nch;
    const long long pe = (units + gridDim.x - 1) / gridDim.x;
    const int first = (int)(((long long)tile * R.nch) / pe);
    const int lastc = (int)(((long long)(tile + 1) * R.nch - 1) / pe);
    const int nseg = lastc - first + 1;
    const int E = t.nrows * nm;                      // valid entries (r, m) -> r * nm + m
    double2* dst = nseg == 1 ? nullptr : part + (size_t)(tile + blockIdx.x) * (WR * WMO);
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      if (i >= cm) break;
#pragma unroll
      for (int j = 0; j < 3; ++j) {
        if (j >= cn) break;
        const int m = 8 * (m_lo + i) + r4;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int r = 8 * (n_lo + j) + 2 * c4 + h;
          if (m < nm && r < t.nrows) {
            const double2 v = make_double2(t1[i][j][h] + t2[i][j][h],
                                           t3[i][j][h] - t1[i][j][h] + t2[i][j][h]);
            if (dst)
              dst[r * nm + m] = v;
            else
              C[(size_t)(t.row0 + r) * a.ldc + m] = v;
          }
        }
      }
    }
    if (nseg > 1) {
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) {
        const unsigned prev = atomicAdd(&counters[tile], 1u);
        last = (prev == (unsigned)nseg - 1);
      }
      __syncthreads();
      if (last) {
        __threadfence();
        const double2* p0 = part + (size_t)(tile + first) * (WR * WMO);
        for (int e = threadIdx.x; e < E; e += NWW * 32) {
          double2 v = make_double2(0.0, 0.0);
          for (int q = 0; q < nseg; q += 4) {   // four slot loads in flight, summed in order
            double2 x4[4];
#pragma unroll
            for (int d = 0; d < 4; ++d)
              x4[d] = q + d < nseg ? __ldcg(&p0[(size_t)(q + d) * (WR * WMO) + e])
                                   : make_double2(0.0, 0.0);
#pragma unroll
            for (int d = 0; d < 4; ++d) v = cadd(v, x4[d]);
          }
          const int r = e / nm, m = e - r * nm;
          C[(size_t)(t.row0 + r) * a.ldc + m] = v;
        }
        if (threadIdx.x == 0) counters[tile] = 0u;
      }
      __syncthreads();
    }
  }
}

// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(kWThreads, 1)
    k_projw_apply(ProjArgs a, const double2* __restrict__ C, const double2* __restrict__ Xin,
                  double2* __restrict__ Y, double ca, double cb, const int* __restrict__ active,
                  int band_mod, int nt_host) {
  pdl_wait();
  extern __shared__ __align__(128) double2 sm[];
  double2* cs = sm + WSA * kWApplyStage;   // C rows of the current tile [WR][kWCs]
  uint64_t* full = reinterpret_cast<uint64_t*>(cs + WR * kWCs);
  uint64_t* empty = full + WSA;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const WRange R = wrange(a, nt_host, KWA);
  if (threadIdx.x == 0) {
    for (int s = 0; s < WSA; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NWW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (R.u0 >= R.u1) return;
  int f_tile = -1, f_k = 0, f_nocc = 0;   // per-tile metadata, fetched once per tile
  auto fill = [&](int u, int s) {         // warp 0, lane 0: the chunk's Phi block
    const int tile = u / R.nch, c = u - tile * R.nch;
    if (tile != f_tile) {
      f_tile = tile;
      f_k = a.tiles[tile].k;
      f_nocc = a.nocc[f_k];
    }
    const uint32_t bytes = (uint32_t)f_nocc * RSWA * 16;
    mbar_expect_tx(&full[s], bytes);
    bulk_g2s(sm + s * kWApplyStage, phiwa_at(a, f_k, f_nocc, c), bytes, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int q = 0; q < WSA && R.u0 + q < R.u1; ++q) fill(R.u0 + q, q);
  const int r4 = lane >> 2, c4 = lane & 3;
  const int wr = w >> 2, wg = w & 3;   // 3 (row groups) x 4 (g fragments of the chunk)
  const bool want_x = ca != 0.0;
  int seq = 0;
  for (int u = R.u0; u < R.u1;) {
    const int tile = u / R.nch;
    const int uend = min(R.u1, (tile + 1) * R.nch);
    const ProjTile t = a.tiles[tile];
    const int nm = a.nocc[t.k];
    __syncthreads();   // every warp is done with the previous tile's C rows
    for (int i = threadIdx.x; i < t.nrows * nm; i += NWW * 32) {
      const int r = i / nm, m = i - r * nm;
      cs[r * kWCs + m] = __ldg(&C[(size_t)(t.row0 + r) * a.ldc + m]);
    }
    int r_lo, r_hi;
    splitn((t.nrows + 7) >> 3, wr, 3, r_lo, r_hi);
    const int cr = r_hi - r_lo;
    int orow[3];
#pragma unroll
    for (int i = 0; i < 3; ++i) {
      const int r = 8 * (r_lo + i) + r4;
      orow[i] = (i < cr && r < t.nrows) ? wxrow(a, t, r) : -1;
      if (orow[i] >= 0 && active && !active[orow[i] % band_mod]) orow[i] = -1;
    }
    __syncthreads();
    for (; u < uend; ++u, ++seq) {
      const size_t g0 = (size_t)(u - tile * R.nch) * KWA + 8 * wg;
      double2 xv[3][2];   // epilogue X values, loaded while the DMMAs run
#pragma unroll
      for (int i = 0; i < 3; ++i)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          xv[i][h] = (want_x && orow[i] >= 0)
                         ? __ldg(&Xin[(size_t)orow[i] * a.nbp + g0 + 2 * c4 + h])
                         : make_double2(0.0, 0.0);
      double t1[3][2], t2[3][2], t3[3][2];
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        t1[i][0] = t1[i][1] = 0.0;
        t2[i][0] = t2[i][1] = 0.0;
        t3[i][0] = t3[i][1] = 0.0;
      }
      const int s = seq % WSA;
      mbar_wait(&full[s], (seq / WSA) & 1);
      const double2* ps = sm + s * kWApplyStage + 8 * wg + r4;
      {
        const double2* ca = cs + (8 * r_lo + r4) * kWCs;
        switch (cr) {   // warp-uniform; see coef_chunk for why the count is a template
          case 1: apply_chunk<1>(ps, ca, nm, c4, t1, t2, t3); break;
          case 2: apply_chunk<2>(ps, ca, nm, c4, t1, t2, t3); break;
          case 3: apply_chunk<3>(ps, ca, nm, c4, t1, t2, t3); break;
          default: break;
        }
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
      if (threadIdx.x == 0 && u + WSA < R.u1) {   // refill once every warp released it
        mbar_wait(&empty[s], (seq / WSA) & 1);
        fill(u + WSA, s);
      }
#pragma unroll
      for (int i = 0; i < 3; ++i) {
        const int row = orow[i];
        if (row < 0) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double dr = t1[i][h] - t2[i][h];
          const double di = t3[i][h] - t1[i][h] - t2[i][h];
          Y[(size_t)row * a.nbp + g0 + 2 * c4 + h] =
              make_double2(ca * xv[i][h].x + cb * dr, ca * xv[i][h].y + cb * di);
        }
      }
    }
  }
}

// ---------------------------------------------------------------------------
static int projw_configure() {
  static bool done = false;
  if (done) return PWB_OK;
  PWB_CUDA(cudaFuncSetAttribute(k_projw_coef, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kWCoefSmem));
  PWB_CUDA(cudaFuncSetAttribute(k_projw_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kWApplySmem));
  done = true;
  return PWB_OK;
}

bool projw_enabled() {
  static const bool off = getenv("PWB_NO_WIDE_PROJ") != nullptr;   // A/B measurement
  return !off;
}

int projw_tiles(const std::vector<int>& row_k, std::vector<ProjTile>& out) {
  out.clear();
  const int n = (int)row_k.size();
  for (int i = 0; i < n;) {
    int j = i;
    while (j < n && row_k[j] == row_k[i] && j - i < WR) ++j;
    out.push_back(ProjTile{i, j - i, row_k[i]});
    i = j;
  }
  return (int)out.size();
}

size_t projw_part_elems(int max_tiles) { return (size_t)(max_tiles + kSM) * WR * WMO; }

// ---- TMA tensor maps of X (2-D FLOAT64 [rows][2 nbp], box 72 rows x 2 RSWC) ----------
static PFN_cuTensorMapEncodeTiled_v12000 tensor_map_encoder() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    (void)cudaGetLastError();
  });
  return fn;
}

// cached per (buffer, rows, nbp): the CG buffers are reused every iteration
static bool x_tensor_maps(const double2* X, long long rows, int nbp, XMaps* out) {
  static thread_local struct Entry {
    const void* p;
    long long rows;
    int nbp;
    XMaps m;
  } cache[32];
  static thread_local int next = 0;
  static const bool off = getenv("PWB_NO_XMAP") != nullptr;   // A/B measurement
  if (off || rows <= 0) return false;
  for (auto& e : cache)
    if (e.p == X && e.rows == rows && e.nbp == nbp) {
      *out = e.m;
      return true;
    }
  auto fn = tensor_map_encoder();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)2 * nbp, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)nbp * 16};
  cuuint32_t es[2] = {1, 1};
  XMaps m;
  for (int h = 0; h < WR / 8; ++h) {
    cuuint32_t box[2] = {(cuuint32_t)(2 * RSWC), (cuuint32_t)(8 * (h + 1))};
    if (fn(&m.m[h], CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, const_cast<double2*>(X), dims, strides,
           box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return false;
  }
  cache[next] = Entry{X, rows, nbp, m};
  next = (next + 1) % 32;
  *out = m;
  return true;
}

int projw_coeffs(const ProjTile* dtiles, int nt_host, int cap, ProjArgs a, const double2* X,
                 double2* part, double2* C, unsigned* counters, cudaStream_t st,
                 long long x_rows) {
  if (cap == 0) return PWB_OK;
  PWB_TRY(projw_configure());
  a.tiles = dtiles;
  const long long units = (long long)cap * (a.nbp / KWC);
  const int grid = (int)std::min<long long>(units, kSM);
  XMaps xmaps;
  memset(&xmaps, 0, sizeof(xmaps));
  const int use_map = x_tensor_maps(X, x_rows, a.nbp, &xmaps) ? 1 : 0;
  (void)launch_k(k_projw_coef, grid, kWThreads, kWCoefSmem, st, a, X, nt_host, part, C,
                 counters, xmaps, use_map);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int projw_apply(const ProjTile* dtiles, int nt_host, int cap, ProjArgs a, const double2* C,
                const double2* Xin, double2* Y, double ca, double cb, const int* active,
                int band_mod, cudaStream_t st) {
  if (cap == 0) return PWB_OK;
  PWB_TRY(projw_configure());
  a.tiles = dtiles;
  const long long units = (long long)cap * (a.nbp / KWA);
  const int grid = (int)std::min<long long>(units, kSM);
  (void)launch_k(k_projw_apply, grid, kWThreads, kWApplySmem, st, a, C, Xin, Y, ca, cb, active,
                 band_mod > 0 ? band_mod : 1, nt_host);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

// chunk-major copy of the orbital rows (one CTA per (orbital row, chunk)): chunk c
// of orbital m of block k at dst + off[k] + (c * nocc[k] + m) * RS, pads zero
template <int KC_, int RS_>
__global__ void k_phiw_chunk(const double2* __restrict__ phi, int nbp, int nk,
                             const int* __restrict__ off, const int* __restrict__ nocc,
                             const int* __restrict__ dst_off, double2* __restrict__ dst) {
  pdl_wait();
  const int b = blockIdx.x, c = blockIdx.y;
  int k = 0;
  while (k + 1 < nk && off[k + 1] <= b) ++k;
  const int m = b - off[k];
  double2* d = dst + dst_off[k] + ((size_t)c * nocc[k] + m) * RS_;
  for (int i = threadIdx.x; i < RS_; i += blockDim.x)
    d[i] = i < KC_ ? phi[(size_t)b * nbp + (size_t)c * KC_ + i] : make_double2(0.0, 0.0);
}

template <int KC_, int RS_>
static int chunk_copy(const double2* phi, int nbp, const std::vector<int>& off_host,
                      const std::vector<int>& nocc_host, DevBuf& buf, DevBuf& d_meta,
                      cudaStream_t st) {
  const int nk = (int)nocc_host.size(), nchunk = nbp / KC_;
  std::vector<int> meta(3 * nk);
  long long tot = 0;
  int nband = 0;
  for (int k = 0; k < nk; ++k) {
    meta[k] = off_host[k];
    meta[nk + k] = nocc_host[k];
    meta[2 * nk + k] = (int)tot;
    tot += (long long)nchunk * nocc_host[k] * RS_;
    nband += nocc_host[k];
  }
  if (tot > 0x7fffffffLL) return fail(PWB_ERR_UNSUPPORTED, "chunk-major orbitals exceed 2^31");
  PWB_TRY(buf.ensure((size_t)std::max<long long>(tot, 1) * sizeof(double2)));
  PWB_TRY(d_meta.ensure(3 * (size_t)nk * sizeof(int)));
  PWB_CUDA(cudaMemcpyAsync(d_meta.ptr, meta.data(), meta.size() * sizeof(int),
                           cudaMemcpyHostToDevice, st));
  const int* dm = as<int>(d_meta);
  if (nband > 0) {
    (void)launch_k(k_phiw_chunk<KC_, RS_>, dim3(nband, nchunk), 64, 0, st, phi, nbp, nk, dm,
                   dm + nk, dm + 2 * nk, as<double2>(buf));
    PWB_LAUNCH_CHECK();
  }
  PWB_CUDA(cudaStreamSynchronize(st));   // meta is a host temporary
  return PWB_OK;
}

int projw_chunked(const double2* phi, int nbp, const std::vector<int>& off_host,
                  const std::vector<int>& nocc_host, DevBuf& phiw, DevBuf& d_meta,
                  DevBuf& phiwa, DevBuf& d_meta_a, cudaStream_t st) {
  if (nbp % KWC || nbp % KWA)
    return fail(PWB_ERR_UNSUPPORTED, "wide projector: row stride not a multiple of 32");
  PWB_TRY((chunk_copy<KWC, RSWC>(phi, nbp, off_host, nocc_host, phiw, d_meta, st)));
  return chunk_copy<KWA, RSWA>(phi, nbp, off_host, nocc_host, phiwa, d_meta_a, st);
}

}  // namespace pwb
