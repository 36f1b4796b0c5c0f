// Device ground state, batched projected Sternheimer PCG, and the chi0 driver.
//
// Reference semantics kept exactly (sternheimer.py:33-98, response.py:110-161):
//   x = 0, r = rhs, z = Q(M^-1 r), p = z, rz = Re<r,z>
//   loop: p = Qp; Ap = Q(Hp - eps p); it++; a = rz/Re<p,Ap> (0 if <= 0);
//         x += a p; r -= a Ap; x = Qx; r = Qr; |r| <= tol -> stop;
//         it >= max_iter -> NonConvergence; z = Q(M^-1 r);
//         b = rz'/rz (0 if rz == 0); p = z + b p
// for every (k, n) row of the batch at once.  Converged rows are masked: their
// x, r, iteration count and residual are frozen exactly where the reference
// loop would have returned, while the remaining rows keep iterating.
#include <cmath>
#include <cstring>
#include <memory>
#include <string>

#include "profile.cuh"
#include "state.cuh"

namespace pwb {

int configure_chi0_kernels(const pwb_grid* g);

// ---- chi0 helpers --------------------------------------------------------------
// delta eps of local rows; fsum = sum w_k f'_n delta eps_n (fixed order, 1 CTA)
__global__ void k_chi0_eps(int r0, int nrows, int ldc, const int* __restrict__ band_k,
                           const int* __restrict__ off, const double2* __restrict__ C,
                           const double* __restrict__ coef, double* __restrict__ deps,
                           double* __restrict__ fsum) {
  pdl_wait();
  // coef layout per band: [0] w*2f/sqrt(Omega), [1] w*f', [2] f', [3] w
  __shared__ double red[256];
  double acc = 0.0;
  for (int i = threadIdx.x; i < nrows; i += 256) {
    const int band = r0 + i;
    const int n = band - off[band_k[band]];
    const double de = C[(size_t)i * ldc + n].x;
    deps[i] = de;
    acc += coef[4 * band + 1] * de;
  }
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int s = 128; s > 0; s >>= 1) {
    if (threadIdx.x < s) red[threadIdx.x] += red[threadIdx.x + s];
    __syncthreads();
  }
  if (threadIdx.x == 0) fsum[0] = red[0];
}

// delta f, accumulation weights, and Cw = W o M for the occupied pair term
__global__ void k_chi0_occ(int r0, int nrows, int ldc, const int* __restrict__ band_k,
                           const int* __restrict__ nocc, const double* __restrict__ coef,
                           const double* __restrict__ fsum, double den, double thresh,
                           const double* __restrict__ deps, const double* __restrict__ wt,
                           const double2* __restrict__ C, double2* __restrict__ Cw,
                           double* __restrict__ c2, double* __restrict__ c1) {
  pdl_wait();
  const int i = blockIdx.x;
  const int band = r0 + i;
  const double def = (fabs(den) > thresh) ? fsum[0] / den : 0.0;
  const int no = nocc[band_k[band]];
  for (int m = threadIdx.x; m < ldc; m += blockDim.x) {
    const double w = (m < no) ? wt[(size_t)band * ldc + m] : 0.0;
    Cw[(size_t)i * ldc + m] = cscale(C[(size_t)i * ldc + m], w);
  }
  if (threadIdx.x == 0) {
    const double df = coef[4 * band + 2] * (deps[i] - def);
    c2[i] = coef[4 * band + 0];
    c1[i] = coef[4 * band + 3] * df;
  }
}

// C(r) = sum_b w_b f'_b |psi_b(r)|^2 over the shard rows (x-fastest output):
// the delta eps_F coefficient of drho, folded in after the sharded all-reduce
__global__ void k_fermi_density(int nx, int nyz, int nband, const double2* __restrict__ psir,
                                const double* __restrict__ coef, int b0, double* __restrict__ out) {
  pdl_wait();
  const long long ng = (long long)nx * nyz;
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;   // x-major index
  if (j >= ng) return;
  double s = 0.0;
  for (int b = 0; b < nband; ++b) {
    const double2 p = psir[(size_t)b * ng + j];
    s += coef[4 * (b0 + b) + 1] * (p.x * p.x + p.y * p.y);
  }
  const int x = (int)(j / nyz), t = (int)(j - (long long)x * nyz);
  out[(size_t)t * nx + x] = s;
}

// packet tail of one rank: [0] sum w f' delta eps (metals), [1] failed rows,
// [2 + b] CG iterations of global row b, [2 + nband + b] residual if row b failed
__global__ void k_pack_tail(int n, int b0, int nband, const int* __restrict__ iters,
                            const double* __restrict__ res, const double* __restrict__ tol,
                            const int* __restrict__ hdr, const double* __restrict__ fsum,
                            int metal, double* __restrict__ tail) {
  pdl_wait();
  __shared__ int nfail;
  if (threadIdx.x == 0) nfail = 0;
  __syncthreads();
  int f = 0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) {
    tail[2 + b0 + i] = (double)iters[i];
    const double r = res[i];
    if (!(r <= tol[i])) {
      tail[2 + nband + b0 + i] = (r == 0.0) ? 1e-300 : r;
      ++f;
    }
  }
  if (f) atomicAdd(&nfail, f);
  __syncthreads();
  if (threadIdx.x == 0) {
    tail[0] = metal ? fsum[0] : 0.0;
    tail[1] = (double)(nfail + (hdr[3] > 0 ? 1 : 0));   // hdr[3] > 0: loop cap reached
  }
}

// drho = sum of partials - delta eps_F C(r), delta eps_F = sum w f' delta eps / sum w f'
__global__ void k_fermi_apply(long long ng, const double* __restrict__ packet, int metal, double den,
                              double* __restrict__ drho) {
  pdl_wait();
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= ng) return;
  double v = packet[i];
  if (metal) v -= (packet[2 * ng] / den) * packet[ng + i];
  drho[i] = v;
}

// psi(r) cache for rows [b0, b1)
static int ensure_psir(pwb_state* st, int b0, int b1) {
  if (st->psir_b0 == b0 && st->psir_b1 == b1) return PWB_OK;
  pwb_grid* g = st->g;
  const int n = b1 - b0;
  PWB_TRY(st->psir.ensure((size_t)std::max(n, 1) * g->ng * sizeof(double2)));
  PWB_TRY(g->wbuf.ensure((size_t)std::max(n, 1) * g->nxa * g->nyz * sizeof(double2)));
  double2* W = as<double2>(g->wbuf);
  const double2* phi = as<double2>(st->phi) + (size_t)b0 * g->nbp;
  const int* bk = as<int>(st->d_band_k) + b0;
  PWB_TRY(launch_plane_inv(g, n, bk, phi, 1.0, W));
  PWB_TRY(launch_pencil_to_cube_xmajor(g, n, W, 1.0 / std::sqrt(g->volume),
                                       as<double2>(st->psir)));
  st->psir_b0 = b0;
  st->psir_b1 = b1;
  return PWB_OK;
}

}  // namespace pwb

using namespace pwb;

extern "C" {

int pwb_state_create(pwb_grid* g, const int* nocc_per_k, const double* kweight,
                     const double* phi, const double* eps, const double* occ,
                     const double* fprime, const double* v_local, const double* rho,
                     pwb_state** out) {
  if (!g || !out) return fail(PWB_ERR_VALUE, "null argument");
  *out = nullptr;
  std::unique_ptr<pwb_state> st(new pwb_state());
  st->g = g;
  st->nk = g->nk;
  st->nocc.assign(nocc_per_k, nocc_per_k + g->nk);
  st->w.assign(kweight, kweight + g->nk);
  st->off.resize(g->nk);
  int nb = 0, ldc = 0;
  for (int k = 0; k < g->nk; ++k) {
    if (st->nocc[k] < 1 || st->nocc[k] > g->nb[k])
      return fail(PWB_ERR_VALUE, "n_occ must lie in 1..n_b for every k");
    st->off[k] = nb;
    nb += st->nocc[k];
    ldc = std::max(ldc, st->nocc[k]);
  }
  st->nband = nb;
  st->ldc = ldc;
  st->eps.assign(eps, eps + nb);
  st->occ.assign(occ, occ + nb);
  st->fprime.assign(fprime, fprime + nb);
  st->band_k.resize(nb);
  double den = 0.0, thr = 0.0;
  for (int k = 0; k < g->nk; ++k) {
    for (int n = 0; n < st->nocc[k]; ++n) {
      st->band_k[st->off[k] + n] = k;
      den += st->w[k] * st->fprime[st->off[k] + n];
    }
    thr += st->w[k] * st->nocc[k];
  }
  st->fp_den = den;
  st->fp_thresh = 1e-14 * thr;   // response.py:135 (abs(fp_sum) > 1e-14 * n_occ)

  // orbitals -> padded rows
  const size_t row = (size_t)g->nbp;
  std::vector<double2> hphi((size_t)nb * row, make_double2(0.0, 0.0));
  const double2* src = reinterpret_cast<const double2*>(phi);
  size_t so = 0;
  for (int k = 0; k < g->nk; ++k)
    for (int n = 0; n < st->nocc[k]; ++n) {
      memcpy(&hphi[(size_t)(st->off[k] + n) * row], src + so, g->nb[k] * sizeof(double2));
      so += g->nb[k];
    }
  PWB_TRY(st->phi.ensure(hphi.size() * sizeof(double2)));
  PWB_CUDA(cudaMemcpy(st->phi.ptr, hphi.data(), hphi.size() * sizeof(double2),
                      cudaMemcpyHostToDevice));
  PWB_TRY(st->d_off.ensure(g->nk * sizeof(int)));
  PWB_TRY(st->d_nocc.ensure(g->nk * sizeof(int)));
  PWB_TRY(st->d_band_k.ensure(nb * sizeof(int)));
  PWB_CUDA(cudaMemcpy(st->d_off.ptr, st->off.data(), g->nk * sizeof(int), cudaMemcpyHostToDevice));
  PWB_CUDA(cudaMemcpy(st->d_nocc.ptr, st->nocc.data(), g->nk * sizeof(int), cudaMemcpyHostToDevice));
  PWB_CUDA(cudaMemcpy(st->d_band_k.ptr, st->band_k.data(), nb * sizeof(int), cudaMemcpyHostToDevice));
  PWB_TRY(proj_chunked(as<double2>(st->phi), g->nbp, st->off, st->nocc, st->phic, st->phic_meta,
                       nullptr));
  st->wide_ok = ldc <= kProjWideOcc && g->nbp % kProjWideChunk == 0;
  if (st->wide_ok)
    PWB_TRY(projw_chunked(as<double2>(st->phi), g->nbp, st->off, st->nocc, st->phiw,
                          st->phiw_meta, st->phiwa, st->phiwa_meta, nullptr));

  // per-band coefficients [w*2f/sqrt(Omega), w*f', f', w]
  std::vector<double> coef(4 * (size_t)nb);
  const double isv = 1.0 / std::sqrt(g->volume);
  for (int b = 0; b < nb; ++b) {
    const double w = st->w[st->band_k[b]];
    coef[4 * b + 0] = w * 2.0 * st->occ[b] * isv;
    coef[4 * b + 1] = w * st->fprime[b];
    coef[4 * b + 2] = st->fprime[b];
    coef[4 * b + 3] = w;
  }
  PWB_TRY(st->d_coef.ensure(coef.size() * sizeof(double)));
  PWB_CUDA(cudaMemcpy(st->d_coef.ptr, coef.data(), coef.size() * sizeof(double),
                      cudaMemcpyHostToDevice));
  // occupied pair weights, stored transposed: wt[band n][m] = W[m][n] (response.py:74-98)
  std::vector<double> wt((size_t)nb * ldc, 0.0);
  for (int k = 0; k < g->nk; ++k) {
    const int o = st->off[k], no = st->nocc[k];
    for (int n = 0; n < no; ++n)
      for (int m = 0; m < no; ++m) {
        if (m == n) continue;
        const double en = st->eps[o + n], em = st->eps[o + m];
        const double fn = st->occ[o + n], fm = st->occ[o + m];
        const double de = en - em;
        const bool degen = std::fabs(de) <= 1e-8 * std::max(1.0, std::fabs(en));
        const double ratio = degen ? st->fprime[o + n] : (fn - fm) / de;
        wt[(size_t)(o + n) * ldc + m] = ratio * fn / (fn * fn + fm * fm);
      }
  }
  PWB_TRY(st->wt.ensure(wt.size() * sizeof(double)));
  PWB_CUDA(cudaMemcpy(st->wt.ptr, wt.data(), wt.size() * sizeof(double), cudaMemcpyHostToDevice));
  PWB_TRY(st->vloc.ensure((size_t)g->ng * sizeof(double)));
  PWB_TRY(st->rho.ensure((size_t)g->ng * sizeof(double)));
  PWB_CUDA(cudaMemcpy(st->vloc.ptr, v_local, (size_t)g->ng * sizeof(double), cudaMemcpyHostToDevice));
  PWB_TRY(st->vloct.ensure((size_t)g->ng * sizeof(double)));
  PWB_TRY(launch_transpose_v(g, as<double>(st->vloc), as<double>(st->vloct)));
  if (rho)
    PWB_CUDA(cudaMemcpy(st->rho.ptr, rho, (size_t)g->ng * sizeof(double), cudaMemcpyHostToDevice));
  else
    PWB_CUDA(cudaMemset(st->rho.ptr, 0, (size_t)g->ng * sizeof(double)));
  PWB_TRY(configure_chi0_kernels(g));
  *out = st.release();
  return PWB_OK;
}

int pwb_state_destroy(pwb_state* st) {
  if (!st) return PWB_OK;
  cudaDeviceSynchronize();
  delete st;   // CgBatch / CgGroup destructors release streams and pinned buffers
  return PWB_OK;
}

int pwb_state_nbands(const pwb_state* st, int* nbands) {
  if (!st || !nbands) return fail(PWB_ERR_VALUE, "null argument");
  *nbands = st->nband;
  return PWB_OK;
}

int pwb_project_out(pwb_state* st, int k, int ncol, double* x) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  if (k < 0 || k >= st->nk) return fail(PWB_ERR_VALUE, "k block out of range");
  if (ncol <= 0) return PWB_OK;
  std::vector<int> key(ncol, k);
  if (st->user_plan_key != key) {
    PWB_TRY(proj_plan(st->user_plan, key, st->nocc, st->g->nbp));
    st->user_plan_key = key;
  }
  size_t pe = proj_part_elems(st->user_plan);
  if (st->wide_ok) pe = std::max(pe, projw_part_elems((int)st->user_plan.wtiles.size()));
  PWB_TRY(st->user_part.ensure(pe * sizeof(double2)));
  PWB_TRY(st->user_cmat.ensure((size_t)ncol * st->ldc * sizeof(double2)));
  return project_rows(st, st->user_plan, reinterpret_cast<double2*>(x), nullptr, ncol, nullptr,
                      as<double2>(st->user_part), as<double2>(st->user_cmat), st->g->stream);
}

int pwb_sternheimer(pwb_state* st, int nrhs, const int* band_host, const double* rhs,
                    const double* tol_host, int max_iter, double* x, int* iters_host,
                    double* res_host) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  if (nrhs <= 0) return PWB_OK;
  std::vector<int> bands(band_host, band_host + nrhs);
  std::vector<double> tol(tol_host, tol_host + nrhs);
  CgBatch& cg = st->cg_user;
  PWB_TRY(cg_setup(st, cg, bands));
  const size_t row = (size_t)st->g->nbp * sizeof(double2);
  PWB_CUDA(cudaMemcpyAsync(cg.rhs.ptr, rhs, nrhs * row, cudaMemcpyDeviceToDevice, st->g->stream));
  int status = cg_solve(st, cg, tol, max_iter, iters_host, res_host);
  PWB_CUDA(cudaMemcpyAsync(x, cg.xr.ptr, nrhs * row, cudaMemcpyDeviceToDevice, st->g->stream));
  PWB_CUDA(cudaStreamSynchronize(st->g->stream));
  return status;
}

int pwb_chi0_begin(pwb_state* st, int b0, int b1, const double* dv, double* fsum) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  if (b0 < 0 || b1 > st->nband || b0 > b1) return fail(PWB_ERR_VALUE, "bad band range");
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  const int n = b1 - b0;
  st->shard_b0 = b0;
  st->shard_b1 = b1;
  std::vector<int> bands(n);
  for (int i = 0; i < n; ++i) bands[i] = b0 + i;
  PWB_TRY(cg_setup(st, st->cg, bands));
  PWB_TRY(ensure_psir(st, b0, b1));
  const size_t row = (size_t)g->nbp * sizeof(double2);
  PWB_TRY(st->dvpsi.ensure(std::max(n, 1) * row));
  PWB_TRY(st->dphi.ensure(std::max(n, 1) * row));
  PWB_TRY(st->cm.ensure((size_t)std::max(n, 1) * st->ldc * sizeof(double2)));
  PWB_TRY(st->cw.ensure((size_t)std::max(n, 1) * st->ldc * sizeof(double2)));
  PWB_TRY(st->scal.ensure((size_t)(3 * std::max(n, 1) + 8) * sizeof(double)));
  if (n == 0) {
    PWB_CUDA(cudaMemsetAsync(fsum, 0, sizeof(double), s));
    return PWB_OK;
  }
  PWB_CUDA(cudaMemsetAsync(st->dvpsi.ptr, 0, n * row, s));
  PWB_CUDA(cudaMemsetAsync(st->dphi.ptr, 0, n * row, s));
  // RHS: dvpsi = to_fourier(dv * to_real(phi_n))  (response.py:127-128)
  PWB_TRY(g->wbuf.ensure((size_t)n * g->nxa * g->nyz * sizeof(double2)));
  double2* W = as<double2>(g->wbuf);
  const double2* phi = as<double2>(st->phi) + (size_t)b0 * g->nbp;
  const int* bk = as<int>(st->d_band_k) + b0;
  double2* dvpsi = as<double2>(st->dvpsi);
  cudaEvent_t er = prof().begin(s);
  PWB_TRY(g->vt.ensure((size_t)g->ng * sizeof(double)));
  PWB_TRY(launch_transpose_v(g, dv, as<double>(g->vt)));
  PWB_TRY(launch_plane_inv(g, n, bk, phi, 1.0, W));
  PWB_TRY(launch_pencil_vmul(g, n, W, as<double>(g->vt), 1.0 / g->ng));
  PWB_TRY(launch_plane_fwd(g, n, bk, W, 1.0, nullptr, nullptr, dvpsi));
  prof().end(PROF_RHS, er, s, n);
  // M^T = (Phi^H dvpsi)^T  (response.py:129)
  ProjArgs a = proj_args(st);
  CgBatch& cg = st->cg;
  PWB_TRY(proj_coeffs_any(st, cg.plan1, a, dvpsi, as<double2>(cg.part), as<double2>(st->cm), s));
  double* deps = as<double>(st->scal);
  (void)launch_k(k_chi0_eps, 1, 256, 0, s, b0, n, st->ldc, as<int>(st->d_band_k), as<int>(st->d_off),
                               as<double2>(st->cm), as<double>(st->d_coef), deps, fsum);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

// Sternheimer solves + accumulation of the pending chi0 into drho.  den /
// thresh decide the Fermi-level shift (response.py:131-136): the state's
// sum_k w_k sum_n f'_n for the full formula, or (0, 1) for delta eps_F = 0
// (the sharded form folds the shift in after the all-reduce).  check = false
// leaves the CG verdict on the device (k_pack_tail reads it) and does not
// synchronise.
static int chi0_finish_impl(pwb_state* st, const double* fsum, double den, double thresh,
                            const double* tol_host, double* drho, int* iters_host, bool check) {
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  const int b0 = st->shard_b0, b1 = st->shard_b1, n = b1 - b0;
  CgBatch& cg = st->cg;
  double* deps = as<double>(st->scal);
  double* c2 = deps + n;
  double* c1 = deps + 2 * n;
  ProjArgs a = proj_args(st);
  (void)launch_k(k_chi0_occ, n, 64, 0, s, b0, n, st->ldc, as<int>(st->d_band_k), as<int>(st->d_nocc),
                              as<double>(st->d_coef), fsum, den, thresh, deps,
                              as<double>(st->wt), as<double2>(st->cm), as<double2>(st->cw), c2,
                              c1);
  PWB_LAUNCH_CHECK();
  // delta phi^P = Phi (W o M)  (response.py:138)
  PWB_TRY(proj_apply_any(st, cg.plan1, a, as<double2>(st->cw), nullptr, as<double2>(st->dphi),
                         0.0, 1.0, nullptr, n, s));
  // rhs = -Q dvpsi (response.py:141), reusing Phi^H dvpsi
  PWB_TRY(proj_apply_any(st, cg.plan1, a, as<double2>(st->cm), as<double2>(st->dvpsi),
                         as<double2>(cg.rhs), -1.0, 1.0, nullptr, n, s));
  std::vector<double> tol(tol_host, tol_host + n);
  // results are read back with the accumulation already queued behind the CG loop
  PWB_TRY(cg_solve(st, cg, tol, -1, nullptr, nullptr, true));
  // drho accumulation (response.py:150-154)
  double2* W = as<double2>(g->wbuf);
  const int* bk = as<int>(st->d_band_k) + b0;
  cudaEvent_t ea = prof().begin(s);
  PWB_TRY(launch_plane_inv2(g, n, bk, as<double2>(st->dphi), as<double2>(cg.xr), W));
  const int ntile = (g->nyz + g->dev.tile - 1) / g->dev.tile;
  int nchunk = std::max(1, std::min(n, (3 * kSM + ntile - 1) / ntile));   // 3 CTAs per SM
  PWB_TRY(st->drho_part.ensure((size_t)nchunk * g->ng * sizeof(double)));
  PWB_TRY(launch_drho_partial(g, n, W, as<double2>(st->psir), c2, c1, nchunk,
                              as<double>(st->drho_part)));
  PWB_TRY(launch_drho_reduce(g, nchunk, as<double>(st->drho_part), drho));
  prof().end(PROF_ACC, ea, s, n);
  if (!check) return PWB_OK;
  PWB_CUDA(cudaStreamSynchronize(s));
  prof().flush();
  return cg_check(cg, tol, iters_host, nullptr);
}

int pwb_chi0_finish(pwb_state* st, const double* fsum, const double* tol_host, double* drho,
                    int* iters_host) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  if (st->shard_b1 == st->shard_b0) {
    PWB_CUDA(cudaMemsetAsync(drho, 0, (size_t)g->ng * sizeof(double), s));
    PWB_CUDA(cudaStreamSynchronize(s));
    return PWB_OK;
  }
  return chi0_finish_impl(st, fsum, st->fp_den, st->fp_thresh, tol_host, drho, iters_host, true);
}

// ---- sharded chi0: one all-reduce per apply ----------------------------------------
static bool is_metal(const pwb_state* st) { return std::fabs(st->fp_den) > st->fp_thresh; }

int pwb_chi0_packet_size(pwb_state* st, long long* n) {
  if (!st || !n) return fail(PWB_ERR_VALUE, "null argument");
  const long long ng = st->g->ng;
  *n = ng * (is_metal(st) ? 2 : 1) + 2 + 2LL * st->nband;
  return PWB_OK;
}

int pwb_chi0_finish_local(pwb_state* st, const double* fsum, const double* tol_host,
                          double* packet) {
  if (!st || !packet) return fail(PWB_ERR_VALUE, "null argument");
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  const int b0 = st->shard_b0, n = st->shard_b1 - b0;
  const size_t ng = g->ng;
  const bool metal = is_metal(st);
  double* tail = packet + ng * (metal ? 2 : 1);
  PWB_CUDA(cudaMemsetAsync(tail, 0, (2 + 2 * (size_t)st->nband) * sizeof(double), s));
  if (n == 0) {
    PWB_CUDA(cudaMemsetAsync(packet, 0, ng * (metal ? 2 : 1) * sizeof(double), s));
    return PWB_OK;
  }
  // delta eps_F = 0 here: the shift is global over all ranks' bands
  PWB_TRY(chi0_finish_impl(st, fsum, 0.0, 1.0, tol_host, packet, nullptr, false));
  if (metal) {
    if (st->fermi_b0 != st->shard_b0 || st->fermi_b1 != st->shard_b1) {
      PWB_TRY(st->fermi_c.ensure(ng * sizeof(double)));
      (void)launch_k(k_fermi_density, (unsigned)((ng + 255) / 256), 256, 0, s, g->nx, g->nyz, n,
                     as<double2>(st->psir), as<double>(st->d_coef), b0, as<double>(st->fermi_c));
      PWB_LAUNCH_CHECK();
      st->fermi_b0 = st->shard_b0;
      st->fermi_b1 = st->shard_b1;
    }
    PWB_CUDA(cudaMemcpyAsync(packet + ng, st->fermi_c.ptr, ng * sizeof(double),
                             cudaMemcpyDeviceToDevice, s));
  }
  CgBatch& cg = st->cg;
  (void)launch_k(k_pack_tail, 1, 256, 0, s, n, b0, st->nband, cg.s.iters, cg.s.res, cg.s.tol,
                 cg.ctl.hdr, fsum, metal ? 1 : 0, tail);
  PWB_LAUNCH_CHECK();
  return PWB_OK;
}

int pwb_chi0_reduce_apply(pwb_state* st, const double* packet, double* drho, int* iters_host,
                          double* residual_host) {
  if (!st || !packet || !drho) return fail(PWB_ERR_VALUE, "null argument");
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  const size_t ng = g->ng;
  const bool metal = is_metal(st);
  const double* tail = packet + ng * (metal ? 2 : 1);
  (void)launch_k(k_fermi_apply, (unsigned)((ng + 255) / 256), 256, 0, s, (long long)ng, packet,
                 metal ? 1 : 0, st->fp_den, drho);
  PWB_LAUNCH_CHECK();
  const size_t nt = 2 + 2 * (size_t)st->nband;
  if (st->h_tail_n < nt) {
    if (st->h_tail) cudaFreeHost(st->h_tail);
    st->h_tail = nullptr;
    PWB_CUDA(cudaMallocHost(&st->h_tail, nt * sizeof(double)));
    st->h_tail_n = nt;
  }
  PWB_CUDA(cudaMemcpyAsync(st->h_tail, tail, nt * sizeof(double), cudaMemcpyDeviceToHost, s));
  PWB_CUDA(cudaStreamSynchronize(s));
  prof().flush();
  const double* t = st->h_tail;
  const int nb = st->nband;
  int first_fail = -1;
  for (int b = 0; b < nb; ++b) {
    const double r = t[2 + nb + b];
    const bool bad = r != 0.0;   // residual of a failed row (NaN included), 0 otherwise
    if (bad && first_fail < 0) first_fail = b;
    if (iters_host) iters_host[b] = bad ? -1 : (int)t[2 + b];
  }
  if (t[1] > 0.0) {
    const double r = first_fail >= 0 ? t[2 + nb + first_fail] : NAN;
    if (residual_host) *residual_host = r;
    set_last_residual(r);
    char buf[256];
    snprintf(buf, sizeof(buf), "Sternheimer CG for band %d stalled at %.3e (%g rows failed "
             "over all ranks)", first_fail, r, t[1]);
    return fail(PWB_ERR_NONCONV, buf);
  }
  return PWB_OK;
}

int pwb_chi0_finish_sharded(pwb_state* st, const double* fsum, const double* tol_host,
                            double* packet, double* drho, int* iters_host, double* residual_host) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  if (!st->comm) return fail(PWB_ERR_CONFIG, "no communicator: call pwb_comm_init first");
  long long n = 0;
  PWB_TRY(pwb_chi0_packet_size(st, &n));
  PWB_TRY(pwb_chi0_finish_local(st, fsum, tol_host, packet));
  PWB_TRY(pwb_allreduce(st, packet, n));
  return pwb_chi0_reduce_apply(st, packet, drho, iters_host, residual_host);
}

int pwb_chi0(pwb_state* st, const double* dv, const double* tol_host, double* drho,
             int* iters_host) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  PWB_TRY(st->fsum.ensure(2 * sizeof(double)));
  PWB_TRY(pwb_chi0_begin(st, 0, st->nband, dv, as<double>(st->fsum)));
  return pwb_chi0_finish(st, as<double>(st->fsum), tol_host, drho, iters_host);
}

int pwb_chi0_host(pwb_state* st, const double* dv_host, const double* tol_host,
                  double* drho_host, int* iters_host) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  pwb_grid* g = st->g;
  PWB_TRY(g->tmp_real.ensure((size_t)2 * g->ng * sizeof(double)));
  double* ddv = as<double>(g->tmp_real);
  double* ddr = ddv + g->ng;
  PWB_CUDA(cudaMemcpyAsync(ddv, dv_host, (size_t)g->ng * sizeof(double), cudaMemcpyHostToDevice,
                           g->stream));
  PWB_TRY(pwb_chi0(st, ddv, tol_host, ddr, iters_host));
  PWB_CUDA(cudaMemcpyAsync(drho_host, ddr, (size_t)g->ng * sizeof(double), cudaMemcpyDeviceToHost,
                           g->stream));
  PWB_CUDA(cudaStreamSynchronize(g->stream));
  return PWB_OK;
}

int pwb_row_norm(pwb_state* st, int k, int real_part, double* out_host) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  if (k < 0 || k >= st->nk) return fail(PWB_ERR_VALUE, "k block out of range");
  pwb_grid* g = st->g;
  const int b0 = st->off[k], n = st->nocc[k];
  DevBuf cache, res;
  PWB_TRY(cache.ensure((size_t)n * g->ng * sizeof(double2)));
  PWB_TRY(res.ensure(sizeof(double)));
  PWB_TRY(g->wbuf.ensure((size_t)n * g->nxa * g->nyz * sizeof(double2)));
  double2* W = as<double2>(g->wbuf);
  PWB_TRY(launch_plane_inv(g, n, as<int>(st->d_band_k) + b0, as<double2>(st->phi) + (size_t)b0 * g->nbp,
                           1.0, W));
  PWB_TRY(launch_pencil_to_cube(g, n, W, 1.0 / std::sqrt(g->volume), as<double2>(cache)));
  PWB_TRY(launch_row_norm(g, n, as<double2>(cache), real_part, as<double>(res)));
  double v = 0.0;
  PWB_CUDA(cudaMemcpyAsync(&v, res.ptr, sizeof(double), cudaMemcpyDeviceToHost, g->stream));
  PWB_CUDA(cudaStreamSynchronize(g->stream));
  *out_host = std::sqrt(v);
  return PWB_OK;
}

}  // extern "C"

extern "C" {

// Q X = X - Phi (Phi^H X) for an arbitrary orthonormal block (no state):
// phi: nocc device rows of length nb; x: ncol device rows of length nb.
int pwb_project_generic(int nb, int nocc, const double* phi, int ncol, double* x) {
  if (nb < 1 || nocc < 1 || ncol < 0) return fail(PWB_ERR_VALUE, "bad projector sizes");
  if (ncol == 0) return PWB_OK;
  static thread_local ProjPlan plan;
  static thread_local DevBuf part, cmat, meta, pphi, px;
  static thread_local std::vector<int> key;
  const int nbp = (nb + 63) / 64 * 64;   // the projector streams rows in 64-coefficient chunks
  std::vector<int> rk(ncol, 0), nocc_v(1, nocc);
  std::vector<int> k2 = {nb, nocc, ncol};
  if (key != k2) {
    PWB_TRY(proj_plan(plan, rk, nocc_v, nbp));
    PWB_TRY(meta.ensure(2 * sizeof(int)));
    int hm[2] = {0, nocc};
    PWB_CUDA(cudaMemcpy(meta.ptr, hm, 2 * sizeof(int), cudaMemcpyHostToDevice));
    key = k2;
  }
  PWB_TRY(part.ensure(proj_part_elems(plan) * sizeof(double2)));
  PWB_TRY(cmat.ensure((size_t)ncol * nocc * sizeof(double2)));
  const double2* P = reinterpret_cast<const double2*>(phi);
  double2* X = reinterpret_cast<double2*>(x);
  double2* XP = X;
  const size_t row = (size_t)nb * sizeof(double2), rowp = (size_t)nbp * sizeof(double2);
  if (nbp != nb) {   // zero-padded copies (pads must be exactly zero)
    PWB_TRY(pphi.ensure((size_t)nocc * rowp));
    PWB_TRY(px.ensure((size_t)ncol * rowp));
    PWB_CUDA(cudaMemsetAsync(pphi.ptr, 0, (size_t)nocc * rowp, nullptr));
    PWB_CUDA(cudaMemsetAsync(px.ptr, 0, (size_t)ncol * rowp, nullptr));
    PWB_CUDA(cudaMemcpy2DAsync(pphi.ptr, rowp, phi, row, row, nocc, cudaMemcpyDeviceToDevice,
                               nullptr));
    PWB_CUDA(cudaMemcpy2DAsync(px.ptr, rowp, x, row, row, ncol, cudaMemcpyDeviceToDevice,
                               nullptr));
    P = as<double2>(pphi);
    XP = as<double2>(px);
  }
  static thread_local DevBuf gphic, gmeta;
  PWB_TRY(proj_chunked(P, nbp, std::vector<int>{0}, std::vector<int>{nocc}, gphic, gmeta, nullptr));
  ProjArgs a;
  a.phic = as<double2>(gphic);
  a.phic_off = as<int>(gmeta) + 2;
  a.phi = P;
  a.off = as<int>(meta);
  a.nocc = as<int>(meta) + 1;
  a.tiles = nullptr;
  a.nbp = nbp;
  a.ldc = nocc;
  a.nrows_total = ncol;
  a.rows = nullptr;
  a.ntiles = nullptr;
  PWB_TRY(proj_coeffs(plan, a, XP, as<double2>(part), as<double2>(cmat), nullptr));
  PWB_TRY(proj_apply(plan, a, as<double2>(cmat), XP, XP, 1.0, -1.0, nullptr, ncol, nullptr));
  if (XP != X)
    PWB_CUDA(cudaMemcpy2DAsync(x, row, XP, rowp, row, ncol, cudaMemcpyDeviceToDevice, nullptr));
  return PWB_OK;   // asynchronous on the legacy default stream
}

int pwb_project_host(int nb, int nocc, const double* phi_host, int ncol, double* x_host) {
  if (nb < 1 || nocc < 1 || ncol < 0) return fail(PWB_ERR_VALUE, "bad projector sizes");
  if (ncol == 0) return PWB_OK;
  DevBuf dphi, dx;
  const size_t bp = (size_t)nocc * nb * sizeof(double2), bx = (size_t)ncol * nb * sizeof(double2);
  PWB_TRY(dphi.ensure(bp));
  PWB_TRY(dx.ensure(bx));
  PWB_CUDA(cudaMemcpy(dphi.ptr, phi_host, bp, cudaMemcpyHostToDevice));
  PWB_CUDA(cudaMemcpy(dx.ptr, x_host, bx, cudaMemcpyHostToDevice));
  PWB_TRY(pwb_project_generic(nb, nocc, as<double>(dphi), ncol, as<double>(dx)));
  PWB_CUDA(cudaMemcpy(x_host, dx.ptr, bx, cudaMemcpyDeviceToHost));
  return PWB_OK;
}

// Pieces of chi0 for a perturbation dv (all bands): diag_host[2*b + {0,1}] =
// <phi_b, dv phi_b> (complex, response.py:53-55) and, if dphi is non-NULL,
// the occupied-subspace response Phi (W o M) as device rows (response.py:101-107).
int pwb_chi0_parts(pwb_state* st, const double* dv, double* diag_host, double* dphi) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  PWB_TRY(st->fsum.ensure(2 * sizeof(double)));
  PWB_TRY(pwb_chi0_begin(st, 0, st->nband, dv, as<double>(st->fsum)));
  pwb_grid* g = st->g;
  cudaStream_t s = g->stream;
  const int n = st->nband;
  std::vector<double2> cm((size_t)n * st->ldc);
  PWB_CUDA(cudaMemcpyAsync(cm.data(), st->cm.ptr, cm.size() * sizeof(double2),
                           cudaMemcpyDeviceToHost, s));
  PWB_CUDA(cudaStreamSynchronize(s));
  for (int b = 0; b < n; ++b) {
    const int m = b - st->off[st->band_k[b]];
    diag_host[2 * b] = cm[(size_t)b * st->ldc + m].x;
    diag_host[2 * b + 1] = cm[(size_t)b * st->ldc + m].y;
  }
  if (dphi) {
    double* deps = as<double>(st->scal);
    (void)launch_k(k_chi0_occ, n, 64, 0, s, 0, n, st->ldc, as<int>(st->d_band_k), as<int>(st->d_nocc),
                                as<double>(st->d_coef), as<double>(st->fsum), st->fp_den,
                                st->fp_thresh, deps, as<double>(st->wt), as<double2>(st->cm),
                                as<double2>(st->cw), deps + n, deps + 2 * n);
    PWB_LAUNCH_CHECK();
    ProjArgs a = proj_args(st);
    PWB_TRY(proj_apply(st->cg.plan1, a, as<double2>(st->cw), nullptr,
                       reinterpret_cast<double2*>(dphi), 0.0, 1.0, nullptr, n, s));
    PWB_CUDA(cudaStreamSynchronize(s));
  }
  return PWB_OK;
}

// orbital_row_norm (response.py:190-199) for arbitrary device sphere rows.
int pwb_row_norm_rows(pwb_grid* g, int nrows, const int* band_k, const double* rows,
                      int real_part, double* out_host) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  DevBuf cache, res;
  PWB_TRY(cache.ensure((size_t)std::max(nrows, 1) * g->ng * sizeof(double2)));
  PWB_TRY(res.ensure(sizeof(double)));
  PWB_TRY(pwb_to_real(g, nrows, band_k, rows, as<double>(cache)));
  PWB_TRY(launch_row_norm(g, nrows, as<double2>(cache), real_part, as<double>(res)));
  double v = 0.0;
  PWB_CUDA(cudaMemcpyAsync(&v, res.ptr, sizeof(double), cudaMemcpyDeviceToHost, g->stream));
  PWB_CUDA(cudaStreamSynchronize(g->stream));
  *out_host = std::sqrt(v);
  return PWB_OK;
}

}  // extern "C"

namespace pwb {
Profiler& prof() {
  static Profiler p;
  return p;
}
}  // namespace pwb

extern "C" {
int pwb_profile_enable(int on) {
  pwb::prof().on = on != 0;
  return PWB_OK;
}
int pwb_profile_reset(void) {
  cudaDeviceSynchronize();
  pwb::prof().flush();
  pwb::prof().reset();
  return PWB_OK;
}
int pwb_profile_read(double* ms, long long* count, long long* units) {
  cudaDeviceSynchronize();
  pwb::prof().flush();
  for (int i = 0; i < pwb::PROF_NCAT; ++i) {
    ms[i] = pwb::prof().ms[i];
    count[i] = pwb::prof().count[i];
    units[i] = pwb::prof().units[i];
  }
  return PWB_OK;
}
int pwb_profile_hist(double* ms, long long* count) {
  cudaDeviceSynchronize();
  pwb::prof().flush();
  for (int i = 0; i < pwb::PROF_NCAT; ++i)
    for (int b = 0; b < pwb::Profiler::NB; ++b) {
      ms[i * pwb::Profiler::NB + b] = pwb::prof().hms[i][b];
      count[i * pwb::Profiler::NB + b] = pwb::prof().hcnt[i][b];
    }
  return PWB_OK;
}
}  // extern "C"
