// Batched projected Sternheimer PCG (reference sternheimer.py:33-98).
//
// Reference semantics kept exactly, per row (one (k, n) pair):
//   x = 0, r = rhs, z = Q(M^-1 r), p = z, rz = Re<r,z>
//   loop: p = Qp; Ap = Q(Hp - eps p); it++; a = rz/Re<p,Ap> (0 if <= 0);
//         x += a p; r -= a Ap; x = Qx; r = Qr; |r| <= tol -> stop;
//         it >= max_iter -> NonConvergence; z = Q(M^-1 r);
//         b = rz'/rz (0 if rz == 0); p = z + b p
// Converged rows are masked: x, r, the iteration count and the residual stay
// exactly where the reference loop returned.
//
// Execution: every iteration starts with a one-CTA compaction kernel that
// turns the device-side active flags into the list of rows still iterating
// and the k-grouped projector tiles.  All later kernels are launched over the
// full batch but blocks beyond the device-side counts exit at once, so one
// iteration is a fixed launch sequence: it is captured once as a CUDA graph
// and replayed (one host call + one 8-byte readback per iteration), and
// converged rows cost no H apply, projector or CG work.
#include <cmath>
#include <cstring>
#include <string>

#include "profile.cuh"
#include "state.cuh"

namespace pwb {

#ifndef PWB_NTC
#define PWB_NTC 1024   // 1024: 11% lower 1-row iteration latency, 2.5% at 261 rows (tools/iter_latency.py)
#endif
constexpr int NTC = PWB_NTC;   // threads per row of the CG vector kernels

__device__ __forceinline__ double block_sum(double v, double* red) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  __syncthreads();
  if (l == 0) red[w] = v;
  __syncthreads();
  double s = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < NTC / 32; ++i) s += red[i];
    red[NTC / 32] = s;
  }
  __syncthreads();
  return red[NTC / 32];
}

__device__ __forceinline__ double minv(const GridDev& g, int k, int s, double pshift) {
  return 1.0 / (g.kin[(size_t)k * g.nbp + s] + pshift);
}

// x = 0, r = rhs, z = M^-1 r
__global__ void __launch_bounds__(NTC) k_cg_init(GridDev g, CgScalars sc, int n,
                                                 const double2* __restrict__ rhs,
                                                 double2* __restrict__ xr, double2* __restrict__ z) {
  pdl_wait();
  const int row = blockIdx.x;
  const int k = sc.row_k[row];
  const double ps = sc.pshift[row];
  double2* x = xr + (size_t)row * g.nbp;
  double2* r = xr + (size_t)(n + row) * g.nbp;
  double2* zz = z + (size_t)row * g.nbp;
  const double2* b = rhs + (size_t)row * g.nbp;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 v = b[s];
    x[s] = make_double2(0.0, 0.0);
    r[s] = v;
    zz[s] = cscale(v, minv(g, k, s, ps));
  }
  if (threadIdx.x == 0) {
    sc.active[row] = 1;
    sc.iters[row] = 0;
    sc.res[row] = 0.0;
  }
}

// rz = Re<r, z>; p = z
__global__ void __launch_bounds__(NTC) k_cg_init2(GridDev g, CgScalars sc, int n,
                                                  const double2* __restrict__ xr,
                                                  const double2* __restrict__ z,
                                                  double2* __restrict__ p, int* __restrict__ hdr,
                                                  int cap) {
  pdl_wait();
  __shared__ double red[NTC / 32 + 1];
  const int row = blockIdx.x;
  if (row == 0 && threadIdx.x == 0) {   // device-side iteration loop: counter and cap
    hdr[4] = 0;   // max_iter failure flag: sticky over the whole solve
    hdr[5] = 0;
    hdr[6] = cap;
  }
  const double2* r = xr + (size_t)(n + row) * g.nbp;
  const double2* zz = z + (size_t)row * g.nbp;
  double2* pp = p + (size_t)row * g.nbp;
  double acc = 0.0;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 a = r[s], c = zz[s];
    acc += a.x * c.x + a.y * c.y;
    pp[s] = c;
  }
  const double rz = block_sum(acc, red);
  if (threadIdx.x == 0) sc.rz[row] = rz;
}

// alpha = rz / Re<p, Ap> (0 if <= 0); x += alpha p; r -= alpha Ap   (active rows)
__global__ void __launch_bounds__(NTC) k_cg_alpha(GridDev g, CgScalars sc, int n,
                                                  const double2* __restrict__ p,
                                                  const double2* __restrict__ ap,
                                                  double2* __restrict__ xr,
                                                  const int* __restrict__ rows,
                                                  const int* __restrict__ nact) {
  pdl_wait();
  __shared__ double red[NTC / 32 + 1];
  if (nact && (int)blockIdx.x >= *nact) return;
  const int row = rows ? rows[blockIdx.x] : blockIdx.x;
  if (!sc.active[row]) return;
  const double2* pp = p + (size_t)row * g.nbp;
  const double2* aa = ap + (size_t)row * g.nbp;
  double acc = 0.0;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 a = pp[s], c = aa[s];
    acc += a.x * c.x + a.y * c.y;
  }
  const double pap = block_sum(acc, red);
  const double alpha = pap > 0.0 ? sc.rz[row] / pap : 0.0;
  double2* x = xr + (size_t)row * g.nbp;
  double2* r = xr + (size_t)(n + row) * g.nbp;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 a = pp[s], c = aa[s];
    double2 xv = x[s], rv = r[s];
    xv.x += alpha * a.x;
    xv.y += alpha * a.y;
    rv.x -= alpha * c.x;
    rv.y -= alpha * c.y;
    x[s] = xv;
    r[s] = rv;
  }
}

// res = |r|; it++; converged / failed masking; z = M^-1 r for rows still active
__global__ void __launch_bounds__(NTC) k_cg_resid(GridDev g, CgScalars sc, int n,
                                                  const double2* __restrict__ xr,
                                                  double2* __restrict__ z,
                                                  const int* __restrict__ rows,
                                                  const int* __restrict__ nact,
                                                  int* __restrict__ counters) {
  pdl_wait();
  __shared__ double red[NTC / 32 + 1];
  if (nact && (int)blockIdx.x >= *nact) return;
  const int row = rows ? rows[blockIdx.x] : blockIdx.x;
  if (!sc.active[row]) return;
  const double2* r = xr + (size_t)(n + row) * g.nbp;
  double acc = 0.0;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 a = r[s];
    acc += a.x * a.x + a.y * a.y;
  }
  const double res = sqrt(block_sum(acc, red));
  const int it = sc.iters[row] + 1;
  const bool done = res <= sc.tol[row];
  const bool failed = !done && it >= sc.maxit[row];
  if (threadIdx.x == 0) {
    sc.res[row] = res;
    sc.iters[row] = it;
    if (done || failed) sc.active[row] = 0;
    if (failed) atomicExch(&counters[1], 1);
    if (!done && !failed) atomicAdd(&counters[0], 1);
  }
  if (done || failed) return;
  const int k = sc.row_k[row];
  const double ps = sc.pshift[row];
  double2* zz = z + (size_t)row * g.nbp;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) zz[s] = cscale(r[s], minv(g, k, s, ps));
}

// rz' = Re<r, z>; beta = rz'/rz (0 if rz == 0); rz = rz'; p = z + beta p
__global__ void __launch_bounds__(NTC) k_cg_beta(GridDev g, CgScalars sc, int n,
                                                 const double2* __restrict__ xr,
                                                 const double2* __restrict__ z,
                                                 double2* __restrict__ p,
                                                 const int* __restrict__ rows,
                                                 const int* __restrict__ nact) {
  pdl_wait();
  __shared__ double red[NTC / 32 + 1];
  if (nact && (int)blockIdx.x >= *nact) return;
  const int row = rows ? rows[blockIdx.x] : blockIdx.x;
  if (!sc.active[row]) return;
  const double2* r = xr + (size_t)(n + row) * g.nbp;
  const double2* zz = z + (size_t)row * g.nbp;
  double acc = 0.0;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 a = r[s], c = zz[s];
    acc += a.x * c.x + a.y * c.y;
  }
  const double rzn = block_sum(acc, red);
  const double rz = sc.rz[row];
  const double beta = rz != 0.0 ? rzn / rz : 0.0;
  double2* pp = p + (size_t)row * g.nbp;
#pragma unroll 4
  for (int s = threadIdx.x; s < g.nbp; s += NTC) {
    const double2 c = zz[s], q = pp[s];
    pp[s] = make_double2(c.x + beta * q.x, c.y + beta * q.y);
  }
  if (threadIdx.x == 0) sc.rz[row] = rzn;
}

// tiles of height T over the stacked span [x rows (c) | r rows (c)] of one k block
__device__ __forceinline__ int stack_tiles(int c, int T) { return 2 * ((c + T - 1) / T); }
__device__ __forceinline__ int merged_tiles(int c, int T) { return (2 * c + T - 1) / T; }
__device__ __forceinline__ void emit_tiles(ProjTile* out, int row0, int c, int T, int k) {
  for (int j = 0; j * T < c; ++j) out[j] = ProjTile{row0 + T * j, min(T, c - T * j), k};
}
__device__ __forceinline__ void emit_stack_tiles(ProjTile* out, int row0, int c, int T, int k) {
  if (merged_tiles(c, T) < stack_tiles(c, T)) {
    emit_tiles(out, row0, 2 * c, T, k);
  } else {
    emit_tiles(out, row0, c, T, k);
    emit_tiles(out + (c + T - 1) / T, row0 + c, c, T, k);
  }
}

// One CTA: active flags -> ascending active-row list, the k-interleaved stacked
// (x; r) list, and the k-grouped projector tiles (<= kProjTileRows rows of one k block).
// Rows are in k-block order, so each k's active rows are contiguous.
__global__ void __launch_bounds__(1024) k_compact(int n, int nk, const int* __restrict__ active,
                                                  const int* __restrict__ row_k, IterCtl ctl) {
  pdl_wait();
  __shared__ int scan[1024];
  __shared__ int kcnt[kMaxK], kstart[kMaxK], ktile[kMaxK], kwide[kMaxK];
  __shared__ int ktile_b[kMaxK], kwide_b[kMaxK];
  __shared__ int carry;
  const int tid = threadIdx.x;
  for (int k = tid; k < nk; k += 1024) kcnt[k] = 0;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (int base = 0; base < n; base += 1024) {
    const int i = base + tid;
    const int f = (i < n && active[i]) ? 1 : 0;
    scan[tid] = f;
    __syncthreads();
    for (int off = 1; off < 1024; off <<= 1) {
      const int v = tid >= off ? scan[tid - off] : 0;
      __syncthreads();
      scan[tid] += v;
      __syncthreads();
    }
    const int pos = carry + scan[tid] - f;
    if (f) {
      ctl.rows[pos] = i;
      atomicAdd(&kcnt[row_k[i]], 1);
    }
    __syncthreads();
    if (tid == 0) carry += scan[1023];
    __syncthreads();
  }
  const int na = carry;
  // The stacked (x; r) list is k-interleaved: block k holds its x rows, then its r
  // rows, so ONE tile can carry both where that saves a tile (c live rows on k:
  // ceil(2c / T) merged tiles against 2 ceil(c / T) separate ones).  In the CG tail,
  // where c <= 8 on most k, the stacked projection then streams each Phi_k once
  // instead of twice and fills DMMA fragments that two 4-row tiles would pad.
  // Where merging saves nothing the x and r spans keep their own tiles (rows
  // consecutive in X: the wide coef kernel loads such a tile with one TMA box copy).
  if (tid == 0) {
    int s = 0, t = 0, wt = 0, tb = 0, wtb = 0;
    for (int k = 0; k < nk; ++k) {
      const int c = kcnt[k];
      kstart[k] = s;
      ktile[k] = t;
      kwide[k] = wt;
      ktile_b[k] = tb;
      kwide_b[k] = wtb;
      s += c;
      t += stack_tiles(c, kProjTileRows) / 2;
      wt += stack_tiles(c, kProjWideRows) / 2;
      tb += min(stack_tiles(c, kProjTileRows), merged_tiles(c, kProjTileRows));
      wtb += min(stack_tiles(c, kProjWideRows), merged_tiles(c, kProjWideRows));
    }
    // one projector path per call: the wide-tile kernels when the live rows fill the
    // wide tiles (>= wide_min rows per tile on average), else the 16-row kernels;
    // the other pair is launched too and exits on its zero count
    const bool wide = ctl.wa != nullptr && wt > 0 && na >= ctl.wide_min * wt;
    const bool wide_b = ctl.wa != nullptr && wtb > 0 && 2 * na >= ctl.wide_min * wtb;
    ctl.hdr[0] = na;
    ctl.hdr[1] = wide ? 0 : t;
    ctl.hdr[2] = wide_b ? 0 : tb;
    ctl.hdr[3] = 0;   // rows still iterating after this iteration (k_cg_resid counts)
    ctl.hdr[8] = wide ? wt : 0;  // wide tiles over rows / over the stacked rows
    ctl.hdr[9] = wide_b ? wtb : 0;
  }
  __syncthreads();
  for (int j = tid; j < na; j += 1024) {
    const int r = ctl.rows[j];
    const int k = row_k[r];
    const int q = 2 * kstart[k] + (j - kstart[k]);
    ctl.rows2[q] = r;
    ctl.rows2[q + kcnt[k]] = r + n;
  }
  for (int k = tid; k < nk; k += 1024) {
    const int c = kcnt[k];
    if (ctl.wa) {
      emit_tiles(ctl.wa + kwide[k], kstart[k], c, kProjWideRows, k);
      emit_stack_tiles(ctl.wb + kwide_b[k], 2 * kstart[k], c, kProjWideRows, k);
    }
    emit_tiles(ctl.ta + ktile[k], kstart[k], c, kProjTileRows, k);
    emit_stack_tiles(ctl.tb + ktile_b[k], 2 * kstart[k], c, kProjTileRows, k);
  }
}

// End of one device-side CG iteration: keep looping while any row still
// iterates (k_cg_resid's count) and the safety cap is not reached.
__global__ void k_loop_ctl(cudaGraphConditionalHandle h, int* __restrict__ hdr) {
  pdl_wait();
  const int n = ++hdr[5];
  cudaGraphSetConditional(h, (hdr[3] > 0 && n < hdr[6]) ? 1u : 0u);
}

CgBatch::~CgBatch() {
  if (h_its) cudaFreeHost(h_its);
  if (h_res) cudaFreeHost(h_res);
  if (exec) cudaGraphExecDestroy(exec);
  if (graph) cudaGraphDestroy(graph);
  if (graph_stream) cudaStreamDestroy(graph_stream);
  if (h_hdr) cudaFreeHost(h_hdr);
}

ProjArgs proj_args(pwb_state* st) {
  ProjArgs a;
  a.phi = as<double2>(st->phi);
  a.off = as<int>(st->d_off);
  a.nocc = as<int>(st->d_nocc);
  a.tiles = nullptr;
  a.nbp = st->g->nbp;
  a.ldc = st->ldc;
  a.nrows_total = 0;
  a.rows = nullptr;
  a.ntiles = nullptr;
  a.phic = as<double2>(st->phic);
  a.phic_off = as<int>(st->phic_meta) + 2 * st->nk;
  a.phiw = st->wide_ok ? as<double2>(st->phiw) : nullptr;
  a.phiw_off = st->wide_ok ? as<int>(st->phiw_meta) + 2 * st->nk : nullptr;
  a.phiwa = st->wide_ok ? as<double2>(st->phiwa) : nullptr;
  a.phiwa_off = st->wide_ok ? as<int>(st->phiwa_meta) + 2 * st->nk : nullptr;
  return a;
}

int projw_min_rows() {
  // Average live rows per wide tile from which the wide-tile kernels run.  Since the
  // inner loops take their fragment counts as template parameters the wide pair wins
  // at every width (tools/qmid.py, configs[4] shape: 1 row on 1 k 30.0 vs 33.8 us,
  // 4 rows on each of 32 k 284 vs 355 us, 16 rows per k 409 vs 433 us), so the 16-row
  // pair only serves states with more than 72 orbitals per k.
  static const int v = getenv("PWB_WIDE_MIN_ROWS") ? atoi(getenv("PWB_WIDE_MIN_ROWS")) : 1;
  return v;
}

// host plans: wide when the rows fill the wide tiles; device plans: the choice is
// made per call by k_compact through the tile counts (both paths are launched)
static bool use_wide(const pwb_state* st, const ProjPlan& pl, const int* ntiles,
                     const int* wntiles) {
  if (!st->wide_ok || !projw_enabled() || plan_wide_tiles(pl) == 0) return false;
  if ((ntiles == nullptr) != (wntiles == nullptr)) return false;
  if (ntiles) return true;
  return pl.nrows >= projw_min_rows() * (int)pl.wtiles.size();
}

int proj_coeffs_any(pwb_state* st, const ProjPlan& pl, ProjArgs a, const double2* X,
                    double2* part, double2* C, cudaStream_t s, const int* wntiles,
                    long long x_rows) {
  if (!use_wide(st, pl, a.ntiles, wntiles)) return proj_coeffs(pl, a, X, part, C, s);
  if (a.ntiles) PWB_TRY(proj_coeffs(pl, a, X, part, C, s));   // exits when wide is chosen
  ProjArgs w = a;
  w.ntiles = wntiles;
  if (x_rows <= 0 && !a.rows && pl.max_tiles == 0 && pl.wmax == 0) x_rows = pl.nrows;
  return projw_coeffs(reinterpret_cast<const ProjTile*>(pl.dwtiles.ptr), (int)pl.wtiles.size(),
                      plan_wide_tiles(pl), w, X, part, C,
                      reinterpret_cast<unsigned*>(pl.wcounters.ptr), s, x_rows);
}

int proj_apply_any(pwb_state* st, const ProjPlan& pl, ProjArgs a, const double2* C,
                   const double2* Xin, double2* Y, double ca, double cb, const int* active,
                   int band_mod, cudaStream_t s, const int* wntiles) {
  if (!use_wide(st, pl, a.ntiles, wntiles))
    return proj_apply(pl, a, C, Xin, Y, ca, cb, active, band_mod, s);
  if (a.ntiles) PWB_TRY(proj_apply(pl, a, C, Xin, Y, ca, cb, active, band_mod, s));
  ProjArgs w = a;
  w.ntiles = wntiles;
  return projw_apply(reinterpret_cast<const ProjTile*>(pl.dwtiles.ptr), (int)pl.wtiles.size(),
                     plan_wide_tiles(pl), w, C, Xin, Y, ca, cb, active, band_mod, s);
}

// Q X in place for the rows of a plan (masked by `active` when given)
int project_rows(pwb_state* st, const ProjPlan& pl, double2* X, const int* active, int band_mod,
                 const int* rows, double2* part, double2* cmat, cudaStream_t s,
                 const int* ntiles, int mult, const int* wntiles) {
  ProjArgs a = proj_args(st);
  a.rows = rows;
  a.ntiles = ntiles;
  cudaEvent_t e = prof().begin(s);
  // host-known tile list with few tiles of one orbital block: the fused
  // single-launch projector (16-80 rows: 15-25% lower latency, tools/qbench.py)
  static const bool no_small = getenv("PWB_NO_SMALLQ") != nullptr;   // A/B measurement
  const int nt = (int)pl.tiles.size();
  if (!no_small && !ntiles && pl.max_tiles == 0 && proj_small_fits(nt, st->g->nbp, st->ldc)) {
    if (st->small_flags.bytes < (size_t)nt * sizeof(unsigned) || !st->small_flags.ptr) {
      PWB_TRY(st->small_flags.ensure((size_t)kSM * sizeof(unsigned)));
      PWB_CUDA(cudaMemset(st->small_flags.ptr, 0, (size_t)kSM * sizeof(unsigned)));
    }
    PWB_TRY(proj_small(pl, a, X, active, band_mod, part, cmat,
                       reinterpret_cast<unsigned*>(st->small_flags.ptr), s));
    prof().end(PROF_Q, e, s, pl.nrows);
    return PWB_OK;
  }
  // rows allocated in X: the CG buffers hold band_mod rows (stacked x; r: 2 band_mod)
  const long long x_rows = ntiles ? (long long)band_mod * mult : pl.nrows;
  PWB_TRY(proj_coeffs_any(st, pl, a, X, part, cmat, s, wntiles, x_rows));
  PWB_TRY(proj_apply_any(st, pl, a, cmat, X, X, 1.0, -1.0, active, band_mod, s, wntiles));
  prof().end(PROF_Q, e, s, prof().rows_hint > 0 ? (long long)mult * prof().rows_hint : pl.nrows);
  return PWB_OK;
}

int cg_setup(pwb_state* st, CgBatch& cg, const std::vector<int>& bands) {
  pwb_grid* g = st->g;
  const int n = (int)bands.size();
  if (cg.nrows == n && cg.bands == bands) return PWB_OK;
  if (st->nk > kMaxK) return fail(PWB_ERR_UNSUPPORTED, "more k-points than kMaxK");
  std::vector<int> rk(n);
  for (int i = 0; i < n; ++i) {
    if (bands[i] < 0 || bands[i] >= st->nband) return fail(PWB_ERR_VALUE, "band index out of range");
    rk[i] = st->band_k[bands[i]];
    if (i > 0 && rk[i] < rk[i - 1])
      return fail(PWB_ERR_VALUE, "Sternheimer rows must be grouped by k in ascending order");
  }
  if (cg.exec) {
    cudaGraphExecDestroy(cg.exec);
    cg.exec = nullptr;
  }
  if (cg.graph) {
    cudaGraphDestroy(cg.graph);
    cg.graph = nullptr;
  }
  cg.nrows = n;
  cg.bands = bands;
  PWB_TRY(proj_plan(cg.plan1, rk, st->nocc, g->nbp));
  // capacity of the device tile lists: every row active
  std::vector<int> per_k(st->nk, 0);
  for (int k : rk) per_k[k]++;
  int maxt = 0, maxocc = 0;
  for (int k = 0; k < st->nk; ++k) {
    maxt += (per_k[k] + kProjTileRows - 1) / kProjTileRows;
    if (per_k[k] > 0) maxocc = std::max(maxocc, st->nocc[k]);
  }
  cg.max_tiles = std::max(1, maxt);
  int maxw = 0;
  for (int k = 0; k < st->nk; ++k) maxw += (per_k[k] + kProjWideRows - 1) / kProjWideRows;
  const int wcap = st->wide_ok ? std::max(1, maxw) : 0;
  PWB_TRY(proj_plan_device(cg.pa, cg.max_tiles, maxocc, g->nbp, wcap));
  PWB_TRY(proj_plan_device(cg.pb, 2 * cg.max_tiles, maxocc, g->nbp, 2 * wcap));
  const size_t row = (size_t)g->nbp * sizeof(double2);
  PWB_TRY(cg.xr.ensure(2 * n * row));
  PWB_TRY(cg.z.ensure(n * row));
  PWB_TRY(cg.p.ensure(n * row));
  PWB_TRY(cg.ap.ensure(n * row));
  PWB_TRY(cg.rhs.ensure(n * row));
  PWB_CUDA(cudaMemset(cg.ap.ptr, 0, n * row));
  PWB_CUDA(cudaMemset(cg.z.ptr, 0, n * row));
  size_t part = std::max({proj_part_elems(cg.plan1), proj_part_elems(cg.pa),
                          proj_part_elems(cg.pb)});
  if (st->wide_ok)
    part = std::max({part, projw_part_elems(2 * wcap), projw_part_elems((int)cg.plan1.wtiles.size())});
  PWB_TRY(cg.part.ensure(part * sizeof(double2)));
  PWB_TRY(cg.cmat.ensure((size_t)2 * n * st->ldc * sizeof(double2)));
  const size_t nd = 5 * (size_t)n, ni = 4 * (size_t)n + 2;
  PWB_TRY(cg.scal.ensure(nd * sizeof(double) + ni * sizeof(int)));
  double* d = as<double>(cg.scal);
  cg.s.rz = d;
  cg.s.res = d + n;
  cg.s.tol = d + 2 * n;
  cg.s.eps = d + 3 * n;
  cg.s.pshift = d + 4 * n;
  int* ip = reinterpret_cast<int*>(d + nd);
  cg.s.active = ip;
  cg.s.iters = ip + n;
  cg.s.maxit = ip + 2 * n;
  cg.s.row_k = ip + 3 * n;
  cg.s.counters = ip + 4 * n;
  PWB_TRY(cg.ctl_buf.ensure((size_t)(kHdrInts + 3 * n) * sizeof(int)));
  cg.ctl.hdr = as<int>(cg.ctl_buf);
  cg.ctl.rows = cg.ctl.hdr + kHdrInts;
  cg.ctl.rows2 = cg.ctl.rows + n;
  cg.ctl.ta = reinterpret_cast<ProjTile*>(cg.pa.dtiles.ptr);
  cg.ctl.tb = reinterpret_cast<ProjTile*>(cg.pb.dtiles.ptr);
  cg.ctl.wa = (wcap > 0 && projw_enabled()) ? reinterpret_cast<ProjTile*>(cg.pa.dwtiles.ptr)
                                             : nullptr;
  cg.ctl.wb = cg.ctl.wa ? reinterpret_cast<ProjTile*>(cg.pb.dwtiles.ptr) : nullptr;
  cg.ctl.wide_min = projw_min_rows();
  std::vector<double> eps(n), ps(n);
  for (int i = 0; i < n; ++i) {
    eps[i] = st->eps[bands[i]];
    ps[i] = std::max(eps[i], 0.1);   // PRECONDITIONER_SHIFT_FLOOR (sternheimer.py:19)
  }
  PWB_CUDA(cudaMemcpy(cg.s.eps, eps.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  PWB_CUDA(cudaMemcpy(cg.s.pshift, ps.data(), n * sizeof(double), cudaMemcpyHostToDevice));
  PWB_CUDA(cudaMemcpy(cg.s.row_k, rk.data(), n * sizeof(int), cudaMemcpyHostToDevice));
  if (!cg.h_hdr) PWB_CUDA(cudaMallocHost(&cg.h_hdr, 8 * sizeof(int)));
  if (!cg.graph_stream) PWB_CUDA(cudaStreamCreateWithFlags(&cg.graph_stream, cudaStreamNonBlocking));
  return PWB_OK;
}

// Enqueue one CG iteration on stream s (direct launches or graph capture).
static int enqueue_iteration(pwb_state* st, CgBatch& cg, cudaStream_t s, bool readback = true) {
  pwb_grid* g = st->g;
  const int n = cg.nrows;
  double2* xr = as<double2>(cg.xr);
  double2* z = as<double2>(cg.z);
  double2* p = as<double2>(cg.p);
  double2* ap = as<double2>(cg.ap);
  double2* part = as<double2>(cg.part);
  double2* cmat = as<double2>(cg.cmat);
  double2* W = as<double2>(g->wbuf);
  const double* vloc = as<double>(st->vloct);   // x-major copy (fused pencil multiply)
  const int* bk = cg.s.row_k;
  const int* nact = cg.ctl.hdr;
  const int* rows = cg.ctl.rows;
  const cudaStream_t saved = g->stream;
  g->stream = s;
  int status = PWB_OK;
  do {
    (void)launch_k(k_compact, 1, 1024, 0, s, n, st->nk, cg.s.active, cg.s.row_k, cg.ctl);
    count_launch();
    if ((status = project_rows(st, cg.pa, p, cg.s.active, n, rows, part, cmat, s, cg.ctl.hdr + 1,
                               1, cg.ctl.hdr + 8)))
      break;
    cudaEvent_t eh = prof().begin(s);
    if ((status = launch_plane_inv(g, n, bk, p, 1.0, W, rows, nact))) break;
    if ((status = launch_pencil_vmul(g, n, W, vloc, 1.0 / g->ng, nact))) break;
    if ((status = launch_plane_fwd(g, n, bk, W, 1.0, p, cg.s.eps, ap, rows, nact))) break;
    prof().end(PROF_H, eh, s, cg.prof_rows);
    if ((status = project_rows(st, cg.pa, ap, cg.s.active, n, rows, part, cmat, s,
                               cg.ctl.hdr + 1, 1, cg.ctl.hdr + 8)))
      break;
    cudaEvent_t ec = prof().begin(s);
    (void)launch_k(k_cg_alpha, n, NTC, 0, s, g->dev, cg.s, n, p, ap, xr, rows, nact);
    count_launch();
    prof().end(PROF_CG, ec, s, cg.prof_rows);
    if ((status = project_rows(st, cg.pb, xr, cg.s.active, n, cg.ctl.rows2, part, cmat, s,
                               cg.ctl.hdr + 2, 2, cg.ctl.hdr + 9)))   // x and r rows together
      break;
    ec = prof().begin(s);
    (void)launch_k(k_cg_resid, n, NTC, 0, s, g->dev, cg.s, n, xr, z, rows, nact, cg.ctl.hdr + 3);
    count_launch();
    prof().end(PROF_CG, ec, s, cg.prof_rows);
    if (readback) cudaMemcpyAsync(cg.h_hdr, cg.ctl.hdr, 8 * sizeof(int), cudaMemcpyDeviceToHost, s);
    if ((status = project_rows(st, cg.pa, z, cg.s.active, n, rows, part, cmat, s, cg.ctl.hdr + 1,
                               1, cg.ctl.hdr + 8)))
      break;
    ec = prof().begin(s);
    (void)launch_k(k_cg_beta, n, NTC, 0, s, g->dev, cg.s, n, xr, z, p, rows, nact);
    count_launch();
    prof().end(PROF_CG, ec, s, cg.prof_rows);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) status = fail(PWB_ERR_CUDA, std::string("CG launch: ") +
                                                          cudaGetErrorString(e));
  } while (false);
  g->stream = saved;
  return status;
}

// launches of one iteration (for the gpu_launches count when replaying the graph)
static unsigned long long g_iter_launches = 0;

// The whole CG loop as ONE graph: a WHILE conditional node whose body is one
// iteration plus k_loop_ctl (no host round trip per iteration).  Returns false
// (nothing built, errors cleared) when the driver refuses it.
static bool build_loop_graph(pwb_state* st, CgBatch& cg) {
  static const bool disabled = getenv("PWB_NO_DEVLOOP") != nullptr;   // A/B measurement
  if (disabled) return false;
  cudaStream_t cs = cg.graph_stream;
  const unsigned long long before = g_launches;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  bool ok = cudaGraphCreate(&graph, 0) == cudaSuccess;
  cudaGraphConditionalHandle h{};
  cudaGraph_t body = nullptr;
  if (ok) ok = cudaGraphConditionalHandleCreate(&h, graph, 1, cudaGraphCondAssignDefault) ==
               cudaSuccess;
  if (ok) {
    cudaGraphNodeParams np = {};
    np.type = cudaGraphNodeTypeConditional;
    np.conditional.handle = h;
    np.conditional.type = cudaGraphCondTypeWhile;
    np.conditional.size = 1;
    cudaGraphNode_t node;
    ok = cudaGraphAddNode(&node, graph, nullptr, 0, &np) == cudaSuccess;
    if (ok) body = np.conditional.phGraph_out[0];
  }
  if (ok) ok = cudaStreamBeginCaptureToGraph(cs, body, nullptr, nullptr, 0,
                                             cudaStreamCaptureModeThreadLocal) == cudaSuccess;
  if (ok) {
    int status = enqueue_iteration(st, cg, cs, false);
    if (status == PWB_OK) {
      (void)launch_k(k_loop_ctl, 1, 1, 0, cs, h, cg.ctl.hdr);
      count_launch();
    }
    cudaGraph_t captured = nullptr;
    const cudaError_t e = cudaStreamEndCapture(cs, &captured);
    ok = status == PWB_OK && e == cudaSuccess;
  }
  if (ok) ok = cudaGraphInstantiate(&exec, graph, 0) == cudaSuccess;
  g_iter_launches = g_launches - before;
  g_launches = before;   // nothing ran during capture
  if (!ok) {
    if (exec) cudaGraphExecDestroy(exec);
    if (graph) cudaGraphDestroy(graph);
    (void)cudaGetLastError();
    return false;
  }
  cg.graph = graph;
  cg.exec = exec;
  cg.loop_graph = true;
  return true;
}

static int ensure_graph(pwb_state* st, CgBatch& cg) {
  if (cg.exec) return PWB_OK;
  if (build_loop_graph(st, cg)) return PWB_OK;
  cg.loop_graph = false;
  cudaStream_t cs = cg.graph_stream;
  const unsigned long long before = g_launches;
  PWB_CUDA(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
  const int status = enqueue_iteration(st, cg, cs);
  cudaGraph_t graph = nullptr;
  const cudaError_t e = cudaStreamEndCapture(cs, &graph);
  if (status != PWB_OK) {
    if (graph) cudaGraphDestroy(graph);
    return status;
  }
  PWB_CUDA(e);
  g_iter_launches = g_launches - before;
  g_launches = before;   // nothing ran during capture
  cg.graph = graph;
  PWB_CUDA(cudaGraphInstantiate(&cg.exec, graph, 0));
  return PWB_OK;
}

// Run the batched PCG on cg.rhs with tolerances tol (host); x = rows [0, n) of cg.xr.
int cg_solve(pwb_state* st, CgBatch& cg, const std::vector<double>& tol, int max_iter,
             int* iters_host, double* res_host, bool defer) {
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  const int n = cg.nrows;
  if (n == 0) return PWB_OK;
  std::vector<int> maxit(n);
  for (int i = 0; i < n; ++i)
    maxit[i] = max_iter > 0 ? max_iter : 10 * g->nb[st->band_k[cg.bands[i]]];
  PWB_CUDA(cudaMemcpyAsync(cg.s.tol, tol.data(), n * sizeof(double), cudaMemcpyHostToDevice, s));
  PWB_CUDA(cudaMemcpyAsync(cg.s.maxit, maxit.data(), n * sizeof(int), cudaMemcpyHostToDevice, s));
  double2* xr = as<double2>(cg.xr);
  double2* z = as<double2>(cg.z);
  double2* p = as<double2>(cg.p);
  (void)launch_k(k_cg_init, n, NTC, 0, s, g->dev, cg.s, n, as<double2>(cg.rhs), xr, z);
  PWB_LAUNCH_CHECK();
  PWB_TRY(project_rows(st, cg.plan1, z, nullptr, n, nullptr, as<double2>(cg.part),
                       as<double2>(cg.cmat), s, nullptr));
  int cap = 0;
  for (int m : maxit) cap = std::max(cap, m);
  (void)launch_k(k_cg_init2, n, NTC, 0, s, g->dev, cg.s, n, xr, z, p, cg.ctl.hdr, cap + 2);
  PWB_LAUNCH_CHECK();
  const size_t wbytes = (size_t)n * g->nxa * g->nyz * sizeof(double2);
  if (g->wbuf.bytes < wbytes || !g->wbuf.ptr) {
    PWB_TRY(g->wbuf.ensure(wbytes));
  }
  if (cg.exec && (cg.graph_w != g->wbuf.ptr || cg.graph_part != cg.part.ptr ||
                  cg.graph_cmat != cg.cmat.ptr)) {   // a captured pointer moved
    cudaGraphExecDestroy(cg.exec);
    cudaGraphDestroy(cg.graph);
    cg.exec = nullptr;
    cg.graph = nullptr;
  }
  const bool use_graph = !prof().on;
  if (use_graph) {
    PWB_TRY(ensure_graph(st, cg));
    cg.graph_w = g->wbuf.ptr;
    cg.graph_part = cg.part.ptr;
    cg.graph_cmat = cg.cmat.ptr;
  }
  cg.prof_rows = n;   // rows active in the next iteration (profiling units only)
  if (cg.h_rows < n) {
    if (cg.h_its) cudaFreeHost(cg.h_its);
    if (cg.h_res) cudaFreeHost(cg.h_res);
    PWB_CUDA(cudaMallocHost(&cg.h_its, (size_t)n * sizeof(int)));
    PWB_CUDA(cudaMallocHost(&cg.h_res, (size_t)n * sizeof(double)));
    cg.h_rows = n;
  }
  cg.loop_ran = use_graph && cg.loop_graph;
  if (cg.loop_ran) {   // the whole loop on the device; results read back with the header
    PWB_CUDA(cudaGraphLaunch(cg.exec, s));
    PWB_CUDA(cudaMemcpyAsync(cg.h_hdr, cg.ctl.hdr, 8 * sizeof(int), cudaMemcpyDeviceToHost, s));
    PWB_CUDA(cudaMemcpyAsync(cg.h_its, cg.s.iters, n * sizeof(int), cudaMemcpyDeviceToHost, s));
    PWB_CUDA(cudaMemcpyAsync(cg.h_res, cg.s.res, n * sizeof(double), cudaMemcpyDeviceToHost, s));
    if (defer) return PWB_OK;
    PWB_CUDA(cudaStreamSynchronize(s));
    return cg_check(cg, tol, iters_host, res_host);
  }
  for (; !(use_graph && cg.loop_graph);) {
    if (use_graph) {
      PWB_CUDA(cudaGraphLaunch(cg.exec, s));
      count_launch((int)g_iter_launches);
    } else {
      prof().rows_hint = cg.prof_rows;
      PWB_TRY(enqueue_iteration(st, cg, s));
    }
    PWB_CUDA(cudaStreamSynchronize(s));
    prof().flush();
    cg.prof_rows = cg.h_hdr[3];
    if (cg.h_hdr[3] == 0) break;   // no row still iterating
  }
  prof().rows_hint = 0;
  PWB_CUDA(cudaMemcpyAsync(cg.h_its, cg.s.iters, n * sizeof(int), cudaMemcpyDeviceToHost, s));
  PWB_CUDA(cudaMemcpyAsync(cg.h_res, cg.s.res, n * sizeof(double), cudaMemcpyDeviceToHost, s));
  if (defer) return PWB_OK;
  PWB_CUDA(cudaStreamSynchronize(s));
  return cg_check(cg, tol, iters_host, res_host);
}

// Verdict of a finished batch from the read-back header and per-row results
// (the stream has been synchronised): reference sternheimer.py:83-90 errors.
int cg_check(CgBatch& cg, const std::vector<double>& tol, int* iters_host, double* res_host) {
  const int n = cg.nrows;
  if (cg.loop_ran) {
    count_launch((int)(g_iter_launches * (unsigned long long)std::max(cg.h_hdr[5], 1)));
    if (cg.h_hdr[3] != 0) return fail(PWB_ERR_NONCONV, "Sternheimer CG: iteration cap reached");
  }
  const bool failed = cg.h_hdr[4] != 0;
  int* its = cg.h_its;
  const double* res = cg.h_res;
  int first_fail = -1;
  for (int i = 0; i < n; ++i) {
    if (!(res[i] <= tol[i])) {   // NaN residuals fail too
      if (first_fail < 0) first_fail = i;
      its[i] = -1;
    }
    if (iters_host) iters_host[i] = its[i];
    if (res_host) res_host[i] = res[i];
  }
  if (failed || first_fail >= 0) {
    set_last_residual(first_fail >= 0 ? res[first_fail] : NAN);
    char buf[256];
    snprintf(buf, sizeof(buf), "Sternheimer CG for band %d stalled at %.3e (target %.3e)",
             first_fail >= 0 ? cg.bands[first_fail] : -1,
             first_fail >= 0 ? res[first_fail] : 0.0, first_fail >= 0 ? tol[first_fail] : 0.0);
    return fail(PWB_ERR_NONCONV, buf);
  }
  return PWB_OK;
}

}  // namespace pwb
