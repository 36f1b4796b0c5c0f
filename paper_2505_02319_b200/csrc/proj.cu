// Occupied-subspace projector Q = 1 - Phi Phi^H as two complex-FP64 GEMMs on
// the FP64 tensor pipe (DMMA: mma.sync.m8n8k4.f64), reference
// sternheimer.py:28-30 and response.py:129,138.
//
//   coef :  C[row][m] = sum_g conj(Phi_k[m][g]) X[row][g]
//           split-K over the sphere; the warps of a CTA reduce in smem, splits
//           are reduced in FIXED split order by the last CTA to finish a tile
//           (threadfence + arrival counter): bitwise reproducible, one launch.
//   apply:  Y[row][g] = a X[row][g] + b sum_m Phi_k[m][g] C[row][m]
//
// Data movement: both kernels are persistent (one CTA per SM) and stream
// their operands through a ring of shared-memory stages filled by TMA bulk
// copies (cp.async.bulk -> UBLKCP, one 1 KB copy per row chunk, completion
// on an mbarrier with expect_tx).  A dedicated producer warp keeps SC
// stages in flight (full/empty mbarrier ring); rows of X are gathered through the
// compacted row list, so active-row compaction costs nothing here.  The
// smem row strides are padded so that the DMMA fragment loads (8 rows x
// 4 consecutive complex) are bank-conflict free.
//
// Padding work is bounded at fragment granularity: a tile of <= 16 rows uses
// ceil(rows/8) n-fragments, an m block of <= 40 orbitals ceil(m/8)
// m-fragments (warp-uniform predicates), so ragged N_occ per k (31..35 at
// BASELINE configs[1]) does not pay for 64-wide blocks.
//
// Complex products use three real DMMAs (Gauss: t1 = a.re b.re, t2 = a.im b.im,
// t3 = (a.re +- a.im)(b.re + b.im)); the combination is formed once per output.
// Measured on B200: DMMA 37.1 TFLOP/s, DFMA 34.0 TFLOP/s (tools/fp64_peak.cu).
#include <cstring>

#include "proj.cuh"
#include "tma.cuh"

namespace pwb {

#ifndef PWB_RED_W
#define PWB_RED_W 1   // modelled cost of one split in the last CTA's sum (1/16 chunk units)
#endif
constexpr int TR = kProjTileRows;   // rows per tile (<= 2 DMMA n-fragments)
constexpr int KC = kProjChunk;      // sphere coefficients per pipeline chunk
constexpr int MF = 5;               // m fragments per block
constexpr int CM = 8 * MF;          // orbitals per block
constexpr int NW = 8;               // warps per CTA
constexpr int SC = 4;               // apply pipeline stages (Phi blocks in flight)
constexpr int SCC = 3;              // coef pipeline stages (X rows + Phi block)
constexpr int RSC = kProjRowStride; // smem / chunk-major row stride (double2): 64 B mod 128 B
constexpr int kCoefStage = (TR + CM) * RSC;   // double2 per coef stage: X rows, Phi block
constexpr int kApplyStage = CM * RSC;         // apply stage: one chunk-major Phi block
constexpr size_t kCoefSmem = (size_t)SCC * kCoefStage * 16 + (size_t)(NW / 2) * CM * TR * 16 + 64;
static_assert(kCoefSmem <= 232448, "stage ring exceeds 227 KB");

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
      : "+d"(d0), "+d"(d1)
      : "d"(a), "d"(b));
}

__device__ __forceinline__ int xrow(const ProjArgs& a, const ProjTile& t, int r) {
  return a.rows ? a.rows[t.row0 + r] : t.row0 + r;
}

// ---------------------------------------------------------------------------
// coef: work item = (tile, m block, split); a split is a run of KC chunks.
struct CoefGeom {
  int ntiles, mtiles, nsplit, split_chunks, nchunk, nitems;
};

// The split count is chosen on the device from the live tile count (it shrinks
// every CG iteration under compaction): the s minimising the modelled time of
// the busiest CTA, in units of 1/16 chunk: items * (chunks + 1 for the item's
// smem/partial reduction) * 16 + s for the last CTA's s-way partial sum.
// (Splitting into single-chunk items looks balanced but measured 6x slower at
// full rows: the per-item reduction dominates.)  Evaluated warp-parallel
// (lane l tries s = l + 1, l + 33, ...) by every warp.
__device__ __forceinline__ CoefGeom coef_geom(const ProjArgs& a, int nt_host, int mtiles,
                                              int smax) {
  CoefGeom g;
  g.ntiles = a.ntiles ? *a.ntiles : nt_host;
  g.mtiles = mtiles;
  g.nchunk = a.nbp / KC;
  const int units = max(1, g.ntiles * mtiles);
  const int lane = threadIdx.x & 31, grid = gridDim.x;
  // entries of one tile's C block: the last CTA's s-way sum costs ~ s E / 132
  // sixteenths of a chunk (qbench at 1..522 rows; 16 rows x 33 orbitals -> 4 s)
  const int E = (g.ntiles == 1 ? a.tiles[0].nrows : TR) * min(CM, a.ldc);
  const int rw = max(PWB_RED_W, E / 132);
  smax = min(smax, g.nchunk);
  unsigned long long best = ~0ull;
  for (int s = lane + 1; s <= smax; s += 32) {
    const int sc = (g.nchunk + s - 1) / s;
    if ((g.nchunk + sc - 1) / sc != s) continue;   // only exact split counts
    const unsigned long long busiest =
        (unsigned long long)((units * s + grid - 1) / grid) * (sc + 1) * 16 + rw * s;
    best = min(best, (busiest << 16) | (unsigned)s);   // ties -> fewer splits
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) best = min(best, __shfl_xor_sync(0xffffffffu, best, o));
  const int s = (int)(best & 0xffff);
  g.split_chunks = (g.nchunk + s - 1) / s;
  g.nsplit = s;
  g.nitems = g.ntiles * mtiles * g.nsplit;
  return g;
}

struct CoefItem {
  ProjTile t;
  int tile, mblk, m0, nm, c0, c1;   // nm orbitals from m0; chunks [c0, c1)
};

__device__ __forceinline__ bool coef_item(const ProjArgs& a, const CoefGeom& g, int item,
                                          CoefItem& it) {
  const int split = item % g.nsplit;
  const int unit = item / g.nsplit;
  it.mblk = unit % g.mtiles;
  it.tile = unit / g.mtiles;
  it.t = a.tiles[it.tile];
  it.m0 = it.mblk * CM;
  it.nm = min(CM, a.nocc[it.t.k] - it.m0);
  it.c0 = split * g.split_chunks;
  it.c1 = min(g.nchunk, it.c0 + g.split_chunks);
  return it.nm > 0 && it.c0 < it.c1 && it.t.nrows > 0;
}

// walks the (item, chunk) sequence of this CTA, skipping empty items
struct CoefCursor {
  int item, chunk;
  CoefItem it;
  bool valid;
  __device__ void first(const ProjArgs& a, const CoefGeom& g) {
    item = blockIdx.x;
    valid = false;
    for (; item < g.nitems; item += gridDim.x)
      if (coef_item(a, g, item, it)) {
        valid = true;
        chunk = it.c0;
        return;
      }
  }
  __device__ void next(const ProjArgs& a, const CoefGeom& g) {
    if (++chunk < it.c1) return;
    valid = false;
    for (item += gridDim.x; item < g.nitems; item += gridDim.x)
      if (coef_item(a, g, item, it)) {
        valid = true;
        chunk = it.c0;
        return;
      }
  }
};

// barrier among the NW consumer warps only (the producer warp runs free)
__device__ __forceinline__ void consumer_sync() {
  asm volatile("bar.sync 1, %0;\n" ::"n"(NW * 32) : "memory");
}

// chunk-major Phi block: orbitals m0 .. m0 + nm - 1 of chunk c of block k
__device__ __forceinline__ const double2* phic_at(const ProjArgs& a, int k, int nocc, int c,
                                                  int m0) {
  return a.phic + a.phic_off[k] + ((size_t)c * nocc + m0) * RSC;
}

// Producer warp (warp NW) of the coef kernel: walks the same (item, chunk)
// sequence as the consumers and keeps SCC stages in flight.  The chunk's Phi
// block is ONE contiguous TMA bulk copy (chunk-major layout); the up to 16
// gathered X rows (1 KB each) are one bulk copy per row issued by lanes
// 0..15, all completing on the stage's mbarrier (one expect_tx arrival).
// (The cp.async 16-byte gather, -DPWB_COEF_CPASYNC, left the consumers
// waiting on the full barrier: 8% slower at 261-522 rows, tools/qbench.py.)
// Row sources are resolved once per item.
__device__ void coef_producer(const ProjArgs& a, const CoefGeom& g, const double2* X,
                              double2* stages, uint64_t* full, uint64_t* empty, int lane) {
  CoefCursor c;
  c.first(a, g);
  int cur = -1, nocc = 0, nrows = 0;
  const double2* xsrc = nullptr;   // row `lane` of the tile (lane < nrows)
  for (unsigned n = 0; c.valid; ++n) {
    const int s = n % SCC;
    if (n >= SCC) mbar_wait(&empty[s], ((n / SCC) + 1) & 1);
    if (c.item != cur) {
      cur = c.item;
      nocc = a.nocc[c.it.t.k];
      nrows = c.it.t.nrows;
      xsrc = lane < nrows ? X + (size_t)xrow(a, c.it.t, lane) * a.nbp : nullptr;
    }
    double2* buf = stages + s * kCoefStage;
    const size_t g0 = (size_t)c.chunk * KC;
#ifndef PWB_COEF_CPASYNC
    if (lane == 0) {   // one arrival: expected bytes of the Phi block and the X rows
      const uint32_t bytes = (uint32_t)c.it.nm * RSC * 16;
      mbar_expect_tx(&full[s], bytes + (uint32_t)nrows * KC * 16);
      bulk_g2s(buf + TR * RSC, phic_at(a, c.it.t.k, nocc, c.chunk, c.it.m0), bytes, &full[s]);
    }
    __syncwarp();
    if (lane < nrows) bulk_g2s(buf + lane * RSC, xsrc + g0, KC * 16, &full[s]);
    c.next(a, g);
    continue;
#endif
    if (lane == 0) {
      const uint32_t bytes = (uint32_t)c.it.nm * RSC * 16;
      mbar_expect_tx(&full[s], bytes);
      bulk_g2s(buf + TR * RSC, phic_at(a, c.it.t.k, nocc, c.chunk, c.it.m0), bytes, &full[s]);
    }
    for (int p = lane; p < nrows * KC; p += 32) {   // 16-byte pieces, row r = p / KC
      const int r = p / KC, o = p - r * KC;
      const double2* src = reinterpret_cast<const double2*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(xsrc), r));
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(su32(buf + r * RSC + o)),
                   "l"(src + g0 + o)
                   : "memory");
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(su32(&full[s]))
                 : "memory");
    c.next(a, g);
  }
}

__global__ void __launch_bounds__((NW + 1) * 32, 1)
    k_proj_coef(ProjArgs a, const double2* __restrict__ X, int nt_host, int tile_cap, int mtiles,
                int smax, double2* __restrict__ part, double2* __restrict__ C,
                unsigned* __restrict__ counters) {
  pdl_wait();
  extern __shared__ __align__(128) double2 sm[];
  double2* stages = sm;
  double2* red = sm + SCC * kCoefStage;   // [NW/2][CM][TR]
  uint64_t* full = reinterpret_cast<uint64_t*>(red + (NW / 2) * CM * TR);
  uint64_t* empty = full + SCC;
  __shared__ bool last;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  const CoefGeom g = coef_geom(a, nt_host, mtiles, smax);
  const size_t stride = (size_t)tile_cap * mtiles * (CM * TR);   // partials per split
  if (threadIdx.x == 0) {
    for (int s = 0; s < SCC; ++s) {
#ifndef PWB_COEF_CPASYNC
      mbar_init(&full[s], 1);        // one expect_tx arrival (all bulk copies)
#else
      mbar_init(&full[s], 1 + 32);   // TMA expect_tx arrival + 32 cp.async lanes
#endif
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (w == NW) {
    coef_producer(a, g, X, stages, full, empty, lane);
    return;
  }
  CoefCursor cons;
  cons.first(a, g);
  // 3-multiplication complex product: t1 = sum pr xr, t2 = sum pi xi,
  // t3 = sum (pr - pi)(xr + xi);  Re = t1 + t2, Im = t3 - t1 + t2
  double t1[MF][2][2], t2[MF][2][2], t3[MF][2][2];
  unsigned seq = 0;
  while (cons.valid) {
    const CoefItem& it = cons.it;
    if (cons.chunk == it.c0) {
#pragma unroll
      for (int ma = 0; ma < MF; ++ma)
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
          t1[ma][nb][0] = t1[ma][nb][1] = 0.0;
          t2[ma][nb][0] = t2[ma][nb][1] = 0.0;
          t3[ma][nb][0] = t3[ma][nb][1] = 0.0;
        }
    }
    const int s = seq % SCC;
    mbar_wait(&full[s], (seq / SCC) & 1);
    const double2* xs = stages + s * kCoefStage;
    const double2* ps = xs + TR * RSC;
    const int nfm = (it.nm + 7) >> 3, nfn = (it.t.nrows + 7) >> 3;
#pragma unroll
    for (int kk = 0; kk < KC / (4 * NW); ++kk) {
      const int gl = 4 * (w + NW * kk) + c4;
      double2 bv[2];
      double bs[2];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        bv[nb] = nb < nfn ? xs[(8 * nb + r4) * RSC + gl] : make_double2(0.0, 0.0);
        bs[nb] = bv[nb].x + bv[nb].y;
      }
      // conj(phi) * x : re = pr xr + pi xi ; im = pr xi - pi xr  (3 real products)
#pragma unroll
      for (int ma = 0; ma < MF; ++ma) {
        if (ma >= nfm) break;
        const double2 av = ps[(8 * ma + r4) * RSC + gl];
        const double ad = av.x - av.y;
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
          if (nb >= nfn) break;
          dmma(t1[ma][nb][0], t1[ma][nb][1], av.x, bv[nb].x);
          dmma(t2[ma][nb][0], t2[ma][nb][1], av.y, bv[nb].y);
          dmma(t3[ma][nb][0], t3[ma][nb][1], ad, bs[nb]);
        }
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);   // this warp is done with stage s
    ++seq;
    if (cons.chunk + 1 >= it.c1) {
      const CoefItem done = it;
      // fixed-order warp reduction in two halves: warp w (< NW/2) adds w + NW/2
      if (w >= NW / 2) {
#pragma unroll
        for (int ma = 0; ma < MF; ++ma)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h)
              red[((w - NW / 2) * CM + 8 * ma + r4) * TR + 8 * nb + 2 * c4 + h] =
                  make_double2(t1[ma][nb][h] + t2[ma][nb][h],
                               t3[ma][nb][h] - t1[ma][nb][h] + t2[ma][nb][h]);
      }
      consumer_sync();
      if (w < NW / 2) {
#pragma unroll
        for (int ma = 0; ma < MF; ++ma)
#pragma unroll
          for (int nb = 0; nb < 2; ++nb)
#pragma unroll
            for (int h = 0; h < 2; ++h) {
              double2& slot = red[(w * CM + 8 * ma + r4) * TR + 8 * nb + 2 * c4 + h];
              slot = make_double2(t1[ma][nb][h] + t2[ma][nb][h] + slot.x,
                                  t3[ma][nb][h] - t1[ma][nb][h] + t2[ma][nb][h] + slot.y);
            }
      }
      consumer_sync();
      const size_t tile_id = (size_t)done.tile * mtiles + done.mblk;
      const int split = done.c0 / g.split_chunks;
      double2* mypart = part + (size_t)split * stride + tile_id * (CM * TR);
      for (int i = threadIdx.x; i < CM * TR; i += NW * 32) {
        const int m = i / TR, r = i - m * TR;
        double2 v = red[i];
#pragma unroll
        for (int q = 1; q < NW / 2; ++q) v = cadd(v, red[q * CM * TR + i]);
        if (g.nsplit == 1) {
          if (r < done.t.nrows && m < done.nm)
            C[(size_t)(done.t.row0 + r) * a.ldc + done.m0 + m] = v;
        } else {
          mypart[i] = v;
        }
      }
      if (g.nsplit > 1) {
        __threadfence();
        consumer_sync();
        if (threadIdx.x == 0) {
          const unsigned prev = atomicAdd(&counters[tile_id], 1u);
          last = (prev == (unsigned)g.nsplit - 1);
        }
        consumer_sync();
        if (last) {
          // Sum the splits of the valid entries in fixed order.  The splits are cut
          // into G contiguous groups summed by different threads (all loads of a
          // group batch in flight together), then the groups are added in order.
          __threadfence();
          const double2* p0 = part + tile_id * (CM * TR);
          const int nr = done.t.nrows;
          const int E = nr * done.nm;   // entry e -> (m = e / nr, r = e % nr)
          const int G = min(NW / 2, (g.nsplit + 7) / 8);
          const int L = (g.nsplit + G - 1) / G;
          for (int j = threadIdx.x; j < G * E; j += NW * 32) {
            const int q = j / E, e = j - q * E;
            const int m = e / nr, i = m * TR + (e - m * nr);
            const int s1 = min(g.nsplit, (q + 1) * L);
            double2 v = make_double2(0.0, 0.0);
            for (int sb = q * L; sb < s1; sb += 8) {
              double2 u[8];
#pragma unroll
              for (int t = 0; t < 8; ++t)
                u[t] = sb + t < s1 ? __ldcg(&p0[(size_t)(sb + t) * stride + i])
                                   : make_double2(0.0, 0.0);
#pragma unroll
              for (int t = 0; t < 8; ++t) v = cadd(v, u[t]);
            }
            red[q * (CM * TR) + i] = v;
          }
          consumer_sync();
          for (int e = threadIdx.x; e < E; e += NW * 32) {
            const int m = e / nr, r = e - m * nr, i = m * TR + r;
            double2 v = red[i];
            for (int q = 1; q < G; ++q) v = cadd(v, red[q * (CM * TR) + i]);
            C[(size_t)(done.t.row0 + r) * a.ldc + done.m0 + m] = v;
          }
          if (threadIdx.x == 0) counters[tile_id] = 0u;
        }
      }
      consumer_sync();   // red / last reused by the next item
    }
    cons.next(a, g);
  }
}

// ---------------------------------------------------------------------------
// apply: work item = (tile, KC chunk of g); each CTA takes a CONTIGUOUS range
// of items (mostly one tile, so C is loaded once per tile run); one stage per
// m block of the item = the chunk's Phi block (one bulk copy).  C rows of the
// current tile live in smem (loaded by the consumers), X values of the
// epilogue are loaded from global one item ahead.  Consumer warp w owns the
// 8 g of fragment w for both row fragments.
struct ApplyCursor {
  int item, item_end, mblk, nchunk, nmb, tile;
  ProjTile t;
  int nocc;
  bool valid;
  __device__ void load(const ProjArgs& a) {
    tile = item / nchunk;
    t = a.tiles[tile];
    nocc = a.nocc[t.k];
    nmb = (nocc + CM - 1) / CM;
  }
  __device__ void first(const ProjArgs& a, int ntiles) {
    nchunk = a.nbp / KC;
    const int nitems = ntiles * nchunk;
    const int per = (nitems + gridDim.x - 1) / gridDim.x;
    item = blockIdx.x * per;
    item_end = min(nitems, item + per);
    mblk = 0;
    valid = item < item_end;
    if (valid) load(a);
  }
  __device__ void next(const ProjArgs& a) {
    if (++mblk < nmb) return;
    mblk = 0;
    ++item;
    valid = item < item_end;
    if (valid) load(a);
  }
};

__device__ void apply_producer(const ProjArgs& a, int ntiles, double2* stages, uint64_t* full,
                               uint64_t* empty, int nst, int lane) {
  ApplyCursor c;
  c.first(a, ntiles);
  for (unsigned n = 0; c.valid; ++n) {
    const int s = n % nst;
    if (n >= (unsigned)nst) mbar_wait(&empty[s], ((n / nst) + 1) & 1);
    if (lane == 0) {
      const int m0 = c.mblk * CM, nm = min(CM, c.nocc - m0);
      const uint32_t bytes = (uint32_t)nm * RSC * 16;
      mbar_expect_tx(&full[s], bytes);
      bulk_g2s(stages + s * kApplyStage, phic_at(a, c.t.k, c.nocc, c.item % c.nchunk, m0), bytes,
               &full[s]);
    }
    __syncwarp();
    c.next(a);
  }
}

__global__ void __launch_bounds__((NW + 1) * 32, 1)
    k_proj_apply(ProjArgs a, const double2* __restrict__ C, const double2* __restrict__ Xin,
                 double2* __restrict__ Y, double ca, double cb, const int* __restrict__ active,
                 int band_mod, int nt_host, int csld, int nst) {
  pdl_wait();
  extern __shared__ __align__(128) double2 sm[];
  double2* cs = sm + nst * kApplyStage;   // C rows of the current tile [TR][csld]
  uint64_t* full = reinterpret_cast<uint64_t*>(cs + TR * csld);
  uint64_t* empty = full + SC;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  const int ntiles = a.ntiles ? *a.ntiles : nt_host;
  const bool want_x = ca != 0.0;
  if (threadIdx.x == 0) {
    for (int s = 0; s < nst; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  if (w == NW) {
    apply_producer(a, ntiles, sm, full, empty, nst, lane);
    return;
  }
  ApplyCursor cons;
  cons.first(a, ntiles);
  int cur_tile = -1;
  int orow[2] = {-1, -1};   // output rows of this lane's fragment rows (-1: skip)
  // 3-multiplication complex product: t1 = sum cr pr, t2 = sum ci pi,
  // t3 = sum (cr + ci)(pr + pi);  Re = t1 - t2, Im = t3 - t1 - t2
  double t1[2][2], t2[2][2], t3[2][2];
  double2 xv[2][2];   // epilogue X values [jb][h] of the current item
  unsigned seq = 0;
  while (cons.valid) {
    if (cons.tile != cur_tile) {   // new tile: C rows -> smem, output rows
      consumer_sync();             // every warp is done with the previous tile's C
      cur_tile = cons.tile;
      const int nr = cons.t.nrows, no = cons.nocc;
      for (int i = threadIdx.x; i < nr * no; i += NW * 32) {
        const int r = i / no, m = i - r * no;
        cs[r * csld + m] = __ldg(&C[(size_t)(cons.t.row0 + r) * a.ldc + m]);
      }
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        const int r = 8 * jb + r4;
        orow[jb] = r < nr ? xrow(a, cons.t, r) : -1;
        if (orow[jb] >= 0 && active && !active[orow[jb] % band_mod]) orow[jb] = -1;
      }
      consumer_sync();
    }
    if (cons.mblk == 0) {
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        t1[jb][0] = t1[jb][1] = 0.0;
        t2[jb][0] = t2[jb][1] = 0.0;
        t3[jb][0] = t3[jb][1] = 0.0;
      }
      const size_t g0 = (size_t)(cons.item % cons.nchunk) * KC;
#pragma unroll
      for (int jb = 0; jb < 2; ++jb)   // in flight during the item's DMMAs
#pragma unroll
        for (int h = 0; h < 2; ++h)
          xv[jb][h] = (want_x && orow[jb] >= 0)
                          ? __ldg(&Xin[(size_t)orow[jb] * a.nbp + g0 + 8 * w + 2 * c4 + h])
                          : make_double2(0.0, 0.0);
    }
    const int s = seq % nst;
    mbar_wait(&full[s], (seq / nst) & 1);
    const double2* ps = sm + s * kApplyStage;
    const int m0 = cons.mblk * CM, nm = min(CM, cons.nocc - m0);
    const int nfn = (cons.t.nrows + 7) >> 3;
#pragma unroll 2
    for (int ms = 0; ms < nm; ms += 4) {
      const int m = ms + c4;
      const bool mok = m < nm;   // contraction index: padding must be exactly zero
      double2 av[2];
#pragma unroll
      for (int jb = 0; jb < 2; ++jb)   // A[j = r4][k = c4] = C[row j][m]
        av[jb] = (mok && jb < nfn) ? cs[(8 * jb + r4) * csld + m0 + m] : make_double2(0.0, 0.0);
      const double2 bv = mok ? ps[m * RSC + 8 * w + r4] : make_double2(0.0, 0.0);   // Phi[m][g]
      const double bs = bv.x + bv.y;
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        if (jb >= nfn) break;
        dmma(t1[jb][0], t1[jb][1], av[jb].x, bv.x);
        dmma(t2[jb][0], t2[jb][1], av[jb].y, bv.y);
        dmma(t3[jb][0], t3[jb][1], av[jb].x + av[jb].y, bs);
      }
    }
    __syncwarp();
    if (lane == 0) mbar_arrive(&empty[s]);
    if (cons.mblk == cons.nmb - 1) {   // epilogue: D fragment row j = r4, g = 2 c4 + {0,1}
      const size_t g0 = (size_t)(cons.item % cons.nchunk) * KC;
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        const int row = orow[jb];
        if (row < 0) continue;
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const double dr = t1[jb][h] - t2[jb][h];
          const double di = t3[jb][h] - t1[jb][h] - t2[jb][h];
          Y[(size_t)row * a.nbp + g0 + 8 * w + 2 * c4 + h] =
              make_double2(ca * xv[jb][h].x + cb * dr, ca * xv[jb][h].y + cb * di);
        }
      }
    }
    ++seq;
    cons.next(a);
  }
}

// ---------------------------------------------------------------------------
// Fused small-batch projector: Q X in ONE launch for a few tiles of one orbital
// block (N_occ <= CM).  CTA (tile t, split j) owns chunks [c0, c1) of tile t:
//   1. one TMA burst brings the X rows and the Phi blocks of ALL its chunks
//      into smem (<= kSmallChunks stages), partial C over them (DMMA, the
//      coef kernel's fragment code), fixed-order warp reduction -> partials;
//   2. the last CTA of tile t to arrive sums the s partials in split order,
//      writes C and bumps the tile's generation flag; the others spin on it
//      (all CTAs are co-resident: grid <= #SM, one CTA per SM by smem);
//   3. every CTA applies Y = X - Phi C on its chunks from the SAME smem copies
//      (no second launch, no reload of X or Phi).
// Latency chain of the two-kernel path at 1-16 rows (~17-24 us per Q:
// two launches, two TMA fills, last-CTA sum, PDL hand-over) -> one launch.
constexpr int kSmallChunks = 3;
constexpr size_t kSmallSmem = (size_t)kSmallChunks * kCoefStage * 16 + (size_t)(NW / 2) * CM * TR * 16 + 64;
static_assert(kSmallSmem <= 232448, "small projector smem");

struct SmallGeom {
  int ntiles, s, sc;
};
__device__ __forceinline__ SmallGeom small_geom(int ntiles, int nchunk) {
  SmallGeom g;
  // as few splits as the smem allows: the split-order sum is the latency
  g.ntiles = ntiles;
  g.sc = kSmallChunks;
  g.s = (nchunk + g.sc - 1) / g.sc;
  return g;
}

__global__ void __launch_bounds__(NW * 32, 1)
    k_proj_small(ProjArgs a, double2* __restrict__ X, const int* __restrict__ active,
                 int band_mod, double2* __restrict__ part, double2* __restrict__ C,
                 unsigned* __restrict__ counters, unsigned* __restrict__ flags, int nt_host) {
  pdl_wait();
  extern __shared__ __align__(128) double2 sm[];
  double2* red = sm + kSmallChunks * kCoefStage;   // [NW/2][CM][TR]; later C tile [TR][CM+4]
  uint64_t* bar = reinterpret_cast<uint64_t*>(red + (NW / 2) * CM * TR);
  __shared__ bool last;
  __shared__ unsigned gen0;
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int r4 = lane >> 2, c4 = lane & 3;
  const int ntiles = a.ntiles ? *a.ntiles : nt_host;
  const int nchunk = a.nbp / KC;
  const SmallGeom gg = small_geom(ntiles, nchunk);
  const int tile = blockIdx.x / gg.s, split = blockIdx.x - tile * gg.s;
  if (tile >= ntiles || gg.sc > kSmallChunks) return;   // (host guarantees sc fits)
  const ProjTile t = a.tiles[tile];
  const int nocc = a.nocc[t.k];
  const int c0 = split * gg.sc, c1 = min(nchunk, c0 + gg.sc), nc = c1 - c0;
  const int nrows = t.nrows;
  if (threadIdx.x == 0) {
    gen0 = *((volatile unsigned*)&flags[tile]);
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();
  // ---- 1. all chunks of this CTA in one TMA burst
  if (w == 0) {
    const uint32_t pb = (uint32_t)nocc * RSC * 16;
    if (lane == 0) mbar_expect_tx(bar, (uint32_t)nc * (pb + (uint32_t)nrows * KC * 16));
    __syncwarp();
    for (int c = 0; c < nc; ++c) {
      double2* buf = sm + c * kCoefStage;
      if (lane == 0) bulk_g2s(buf + TR * RSC, phic_at(a, t.k, nocc, c0 + c, 0), pb, bar);
      if (lane < nrows)
        bulk_g2s(buf + lane * RSC, X + (size_t)xrow(a, t, lane) * a.nbp + (size_t)(c0 + c) * KC,
                 KC * 16, bar);
    }
  }
  // zero the unused tails of the stages (rows >= nrows, orbitals >= nocc) are
  // never read: the fragment predicates below bound rows / orbitals
  mbar_wait(bar, 0);
  const int nfm = (nocc + 7) >> 3, nfn = (nrows + 7) >> 3;
  double t1[MF][2][2], t2[MF][2][2], t3[MF][2][2];
#pragma unroll
  for (int ma = 0; ma < MF; ++ma)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      t1[ma][nb][0] = t1[ma][nb][1] = 0.0;
      t2[ma][nb][0] = t2[ma][nb][1] = 0.0;
      t3[ma][nb][0] = t3[ma][nb][1] = 0.0;
    }
  for (int c = 0; c < nc; ++c) {
    const double2* xs = sm + c * kCoefStage;
    const double2* ps = xs + TR * RSC;
#pragma unroll
    for (int kk = 0; kk < KC / (4 * NW); ++kk) {
      const int gl = 4 * (w + NW * kk) + c4;
      double2 bv[2];
      double bs[2];
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        bv[nb] = (nb < nfn && 8 * nb + r4 < nrows) ? xs[(8 * nb + r4) * RSC + gl]
                                                    : make_double2(0.0, 0.0);
        bs[nb] = bv[nb].x + bv[nb].y;
      }
#pragma unroll
      for (int ma = 0; ma < MF; ++ma) {
        if (ma >= nfm) break;
        const double2 av = (8 * ma + r4 < nocc) ? ps[(8 * ma + r4) * RSC + gl]
                                                 : make_double2(0.0, 0.0);
        const double ad = av.x - av.y;
#pragma unroll
        for (int nb = 0; nb < 2; ++nb) {
          if (nb >= nfn) break;
          dmma(t1[ma][nb][0], t1[ma][nb][1], av.x, bv[nb].x);
          dmma(t2[ma][nb][0], t2[ma][nb][1], av.y, bv[nb].y);
          dmma(t3[ma][nb][0], t3[ma][nb][1], ad, bs[nb]);
        }
      }
    }
  }
  // fixed-order warp reduction (as in k_proj_coef)
  if (w >= NW / 2) {
#pragma unroll
    for (int ma = 0; ma < MF; ++ma)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h)
          red[((w - NW / 2) * CM + 8 * ma + r4) * TR + 8 * nb + 2 * c4 + h] =
              make_double2(t1[ma][nb][h] + t2[ma][nb][h], t3[ma][nb][h] - t1[ma][nb][h] + t2[ma][nb][h]);
  }
  __syncthreads();
  if (w < NW / 2) {
#pragma unroll
    for (int ma = 0; ma < MF; ++ma)
#pragma unroll
      for (int nb = 0; nb < 2; ++nb)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          double2& slot = red[(w * CM + 8 * ma + r4) * TR + 8 * nb + 2 * c4 + h];
          slot = make_double2(t1[ma][nb][h] + t2[ma][nb][h] + slot.x,
                              t3[ma][nb][h] - t1[ma][nb][h] + t2[ma][nb][h] + slot.y);
        }
  }
  __syncthreads();
  double2* mypart = part + ((size_t)tile * gg.s + split) * (CM * TR);
  for (int i = threadIdx.x; i < CM * TR; i += NW * 32) {
    double2 v = red[i];
#pragma unroll
    for (int q = 1; q < NW / 2; ++q) v = cadd(v, red[q * CM * TR + i]);
    mypart[i] = v;
  }
  // ---- 2. last CTA of the tile: fixed split-order sum -> C, then release the tile
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&counters[tile], 1u) == (unsigned)gg.s - 1;
  __syncthreads();
  const int E = nrows * nocc;
  if (last) {
    __threadfence();
    // G groups of consecutive splits per entry (all their loads in flight),
    // then the groups in order: fixed summation order for given (s, E)
    const double2* p0 = part + (size_t)tile * gg.s * (CM * TR);
    const int G = max(1, min(NW / 2, (NW * 32) / max(E, 1)));
    const int L = (gg.s + G - 1) / G;
    for (int j = threadIdx.x; j < G * E; j += NW * 32) {
      const int q = j / E, e = j - q * E;
      const int m = e / nrows, i = m * TR + (e - m * nrows);
      const int s1 = min(gg.s, (q + 1) * L);
      double2 v = make_double2(0.0, 0.0);
      for (int sb = q * L; sb < s1; sb += 8) {
        double2 u[8];
#pragma unroll
        for (int qq = 0; qq < 8; ++qq)
          u[qq] = sb + qq < s1 ? __ldcg(&p0[(size_t)(sb + qq) * (CM * TR) + i])
                               : make_double2(0.0, 0.0);
#pragma unroll
        for (int qq = 0; qq < 8; ++qq) v = cadd(v, u[qq]);
      }
      red[q * (CM * TR) + i] = v;
    }
    __syncthreads();
    for (int e = threadIdx.x; e < E; e += NW * 32) {
      const int m = e / nrows, r = e - m * nrows, i = m * TR + r;
      double2 v = red[i];
      for (int q = 1; q < G; ++q) v = cadd(v, red[q * (CM * TR) + i]);
      C[(size_t)(t.row0 + r) * a.ldc + m] = v;
    }
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
      counters[tile] = 0u;
      atomicAdd(&flags[tile], 1u);   // publishes C of this tile
    }
  } else if (threadIdx.x == 0) {
    while (*((volatile unsigned*)&flags[tile]) == gen0) __nanosleep(64);
  }
  __syncthreads();
  __threadfence();
  // ---- 3. Y = X - Phi C on this CTA's chunks, from the smem copies
  constexpr int CS = CM + 4;   // C tile stride (4 mod 8: conflict-free fragment loads)
  double2* cs = red;           // reuse: [TR][CS]
  for (int e = threadIdx.x; e < TR * CS; e += NW * 32) {
    const int r = e / CS, m = e - r * CS;
    cs[e] = (r < nrows && m < nocc) ? __ldcg(&C[(size_t)(t.row0 + r) * a.ldc + m])
                                    : make_double2(0.0, 0.0);
  }
  __syncthreads();
  int orow[2];
#pragma unroll
  for (int jb = 0; jb < 2; ++jb) {
    const int r = 8 * jb + r4;
    orow[jb] = r < nrows ? xrow(a, t, r) : -1;
    if (orow[jb] >= 0 && active && !active[orow[jb] % band_mod]) orow[jb] = -1;
  }
  for (int c = 0; c < nc; ++c) {
    const double2* xs = sm + c * kCoefStage;
    const double2* ps = xs + TR * RSC;
    double u1[2][2] = {}, u2[2][2] = {}, u3[2][2] = {};
    for (int ms = 0; ms < nocc; ms += 4) {
      const int m = ms + c4;
      const bool mok = m < nocc;
      double2 av[2];
#pragma unroll
      for (int jb = 0; jb < 2; ++jb)   // A[j = r4][k = c4] = C[row j][m]
        av[jb] = (mok && jb < nfn) ? cs[(8 * jb + r4) * CS + m] : make_double2(0.0, 0.0);
      const double2 bv = mok ? ps[m * RSC + 8 * w + r4] : make_double2(0.0, 0.0);   // Phi[m][g]
      const double bsum = bv.x + bv.y;
#pragma unroll
      for (int jb = 0; jb < 2; ++jb) {
        if (jb >= nfn) break;
        dmma(u1[jb][0], u1[jb][1], av[jb].x, bv.x);
        dmma(u2[jb][0], u2[jb][1], av[jb].y, bv.y);
        dmma(u3[jb][0], u3[jb][1], av[jb].x + av[jb].y, bsum);
      }
    }
    const size_t g0 = (size_t)(c0 + c) * KC;
#pragma unroll
    for (int jb = 0; jb < 2; ++jb) {
      const int row = orow[jb];
      if (row < 0) continue;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gl = 8 * w + 2 * c4 + h;
        const double2 x = xs[(8 * jb + r4) * RSC + gl];
        const double dr = u1[jb][h] - u2[jb][h];
        const double di = u3[jb][h] - u1[jb][h] - u2[jb][h];
        X[(size_t)row * a.nbp + g0 + gl] = make_double2(x.x - dr, x.y - di);
      }
    }
  }
}

int proj_small(const ProjPlan& pl, ProjArgs a, double2* X, const int* active, int band_mod,
               double2* part, double2* C, unsigned* flags, cudaStream_t st) {
  const int cap = plan_tiles(pl);
  if (cap == 0) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  (void)launch_k(k_proj_small, kSM, NW * 32, kSmallSmem, st, a, X, active,
                 band_mod > 0 ? band_mod : 1, part, C,
                 reinterpret_cast<unsigned*>(pl.counters.ptr), flags, (int)pl.tiles.size());
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

bool proj_small_fits(int ntiles, int nbp, int maxocc) {
  if (maxocc > CM || ntiles <= 0 || ntiles > kSM) return false;
  const int nchunk = nbp / KC;
  const int s = (nchunk + kSmallChunks - 1) / kSmallChunks;
  return (long)s * ntiles <= kSM;
}

// ---------------------------------------------------------------------------
static int proj_configure() {
  static bool done = false;
  if (done) return PWB_OK;
  PWB_CUDA(cudaFuncSetAttribute(k_proj_coef, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kCoefSmem));
  PWB_CUDA(cudaFuncSetAttribute(k_proj_small, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                (int)kSmallSmem));
  PWB_CUDA(cudaFuncSetAttribute(k_proj_apply, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                232448));
  done = true;
  return PWB_OK;
}

static int nsplit_max(int nbp) { return std::max(1, std::min(kSM, nbp / KC)); }

int proj_plan(ProjPlan& pl, const std::vector<int>& row_k, const std::vector<int>& nocc,
              int nbp, cudaStream_t st, bool async) {
  PWB_TRY(proj_configure());
  if (nbp % KC) return fail(PWB_ERR_UNSUPPORTED, "projector: row stride not a multiple of 64");
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
  pl.wmax = 0;
  projw_tiles(row_k, pl.wtiles);
  if (!pl.wtiles.empty()) {   // wide list: small, uploaded synchronously
    const size_t nw = pl.wtiles.size();
    if (pl.dwtiles.bytes < nw * sizeof(ProjTile) || !pl.dwtiles.ptr)
      PWB_TRY(pl.dwtiles.ensure(nw * sizeof(ProjTile)));
    if (async) {
      PWB_CUDA(cudaStreamSynchronize(st));
    }
    PWB_CUDA(cudaMemcpy(pl.dwtiles.ptr, pl.wtiles.data(), nw * sizeof(ProjTile),
                        cudaMemcpyHostToDevice));
    if (pl.wcounters.bytes < nw * sizeof(unsigned) || !pl.wcounters.ptr) {
      PWB_TRY(pl.wcounters.ensure(nw * sizeof(unsigned)));
      PWB_CUDA(cudaMemset(pl.wcounters.ptr, 0, nw * sizeof(unsigned)));
    }
  }
  pl.nsplit = nsplit_max(nbp);   // upper bound; the live count is chosen on the device
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

int proj_plan_device(ProjPlan& pl, int max_tiles, int maxocc, int nbp, int wide_tiles) {
  PWB_TRY(proj_configure());
  if (nbp % KC) return fail(PWB_ERR_UNSUPPORTED, "projector: row stride not a multiple of 64");
  pl.tiles.clear();
  pl.wtiles.clear();
  pl.wmax = wide_tiles;
  if (wide_tiles > 0) {
    PWB_TRY(pl.dwtiles.ensure((size_t)wide_tiles * sizeof(ProjTile)));
    PWB_TRY(pl.wcounters.ensure((size_t)wide_tiles * sizeof(unsigned)));
    PWB_CUDA(cudaMemset(pl.wcounters.ptr, 0, (size_t)wide_tiles * sizeof(unsigned)));
  }
  pl.max_tiles = max_tiles;
  pl.nrows = max_tiles * TR;
  pl.mtiles = std::max(1, (maxocc + CM - 1) / CM);
  pl.nsplit = nsplit_max(nbp);
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
  const int grid = (int)std::min<long>(items, kSM);
  (void)launch_k(k_proj_coef, grid, (NW + 1) * 32, kCoefSmem, st, a, X, (int)pl.tiles.size(), cap, pl.mtiles,
                                                pl.nsplit, part, C,
                                                reinterpret_cast<unsigned*>(pl.counters.ptr));
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int proj_apply(const ProjPlan& pl, ProjArgs a, const double2* C, const double2* Xin, double2* Y,
               double ca, double cb, const int* active, int band_mod, cudaStream_t st) {
  const int cap = plan_tiles(pl);
  if (cap == 0) return PWB_OK;
  a.tiles = reinterpret_cast<const ProjTile*>(pl.dtiles.ptr);
  a.nrows_total = pl.nrows;
  const long items = (long)cap * (a.nbp / KC);
  const int grid = (int)std::min<long>(items, kSM);
  const int csld = ((a.ldc + 3) / 8) * 8 + 4;   // C rows in smem: stride = 4 mod 8 (conflict-free)
  int nst = SC;   // fewer Phi stages in flight when many orbitals' C rows take the smem
  while (nst > 2 && (size_t)nst * kApplyStage * 16 + (size_t)TR * csld * 16 + 64 > 232448) --nst;
  const size_t smem = (size_t)nst * kApplyStage * 16 + (size_t)TR * csld * 16 + 64;
  if (smem > 232448) return fail(PWB_ERR_UNSUPPORTED, "projector: too many orbitals per k");
  (void)launch_k(k_proj_apply, grid, (NW + 1) * 32, smem, st, a, C, Xin, Y, ca, cb, active,
                 band_mod > 0 ? band_mod : 1, (int)pl.tiles.size(), csld, nst);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

// ---------------------------------------------------------------------------
// chunk-major copy of the orbital rows (one CTA per (orbital row, chunk))
__global__ void k_phi_chunk(const double2* __restrict__ phi, int nbp, int nk,
                            const int* __restrict__ off, const int* __restrict__ nocc,
                            const int* __restrict__ phic_off, double2* __restrict__ phic) {
  pdl_wait();
  const int b = blockIdx.x, c = blockIdx.y;
  int k = 0;
  while (k + 1 < nk && off[k + 1] <= b) ++k;
  const int m = b - off[k];
  double2* dst = phic + phic_off[k] + ((size_t)c * nocc[k] + m) * RSC;
  for (int i = threadIdx.x; i < RSC; i += blockDim.x)
    dst[i] = i < KC ? phi[(size_t)b * nbp + (size_t)c * KC + i] : make_double2(0.0, 0.0);
}

int proj_chunked(const double2* phi, int nbp, const std::vector<int>& off_host,
                 const std::vector<int>& nocc_host, DevBuf& phic, DevBuf& d_phic_off,
                 cudaStream_t st) {
  if (nbp % KC) return fail(PWB_ERR_UNSUPPORTED, "projector: row stride not a multiple of 64");
  const int nk = (int)nocc_host.size(), nchunk = nbp / KC;
  std::vector<int> po(nk), meta(3 * nk);
  long long tot = 0;
  int nband = 0;
  for (int k = 0; k < nk; ++k) {
    po[k] = (int)tot;
    tot += (long long)nchunk * nocc_host[k] * RSC;
    nband += nocc_host[k];
  }
  if (tot > 0x7fffffffLL) return fail(PWB_ERR_UNSUPPORTED, "chunk-major orbitals exceed 2^31");
  for (int k = 0; k < nk; ++k) {
    meta[k] = off_host[k];
    meta[nk + k] = nocc_host[k];
    meta[2 * nk + k] = po[k];
  }
  PWB_TRY(phic.ensure((size_t)std::max<long long>(tot, 1) * sizeof(double2)));
  PWB_TRY(d_phic_off.ensure(3 * (size_t)nk * sizeof(int)));
  PWB_CUDA(cudaMemcpyAsync(d_phic_off.ptr, meta.data(), meta.size() * sizeof(int),
                           cudaMemcpyHostToDevice, st));
  const int* dm = as<int>(d_phic_off);
  if (nband > 0) {
    (void)launch_k(k_phi_chunk, dim3(nband, nchunk), 64, 0, st, phi, nbp, nk, dm, dm + nk,
                   dm + 2 * nk, as<double2>(phic));
    PWB_LAUNCH_CHECK();
  }
  PWB_CUDA(cudaStreamSynchronize(st));   // meta is a host temporary
  return PWB_OK;
}

}  // namespace pwb
