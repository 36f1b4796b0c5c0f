// Device-resident ground state and the batched Sternheimer / chi0 runtime.
#pragma once

#include <vector>

#include "grid.cuh"
#include "proj.cuh"

namespace pwb {

// per-row CG scalars (struct of arrays, device)
struct CgScalars {
  double* rz;
  double* res;
  double* tol;
  double* eps;     // eigenvalue shift (H - eps)
  double* pshift;  // max(eps, 0.1): kinetic preconditioner shift
  int* active;
  int* iters;
  int* maxit;
  int* row_k;
  int* counters;   // [0] active count, [1] failure flag
};

struct CgBatch {
  int nrows = 0;
  std::vector<int> bands;   // global band of each row
  ProjPlan plan1;           // rows [0, n)
  ProjPlan plan2;           // rows [0, 2n) for the stacked (x; r) buffer
  DevBuf xr, z, p, ap, rhs;
  DevBuf scal;              // CgScalars storage
  DevBuf part, cmat;        // GEMM scratch
  CgScalars s;
  int* h_counters = nullptr;  // pinned
  // active-row compaction (rebuilt every CG iteration)
  int* h_active = nullptr;    // pinned copy of s.active
  int* h_rows = nullptr;      // pinned: [na active rows][na rows][na rows + n]
  DevBuf d_rows;
  ProjPlan plan_a, plan_b;
};

// accumulation kernels (chi0.cu)
int launch_drho_partial(pwb_grid* g, int nband, const double2* W, const double2* psir,
                        const double* c2, const double* c1, int nchunk, double* partial);
int launch_drho_reduce(pwb_grid* g, int nchunk, const double* partial, double* drho);
int launch_row_norm(pwb_grid* g, int nband, const double2* psir, int real_part, double* out);

}  // namespace pwb

struct pwb_state {
  pwb_grid* g = nullptr;
  int nk = 0, nband = 0, ldc = 0;
  std::vector<int> nocc, off, band_k;
  std::vector<double> w, eps, occ, fprime;
  double fp_den = 0.0;       // sum_k w_k sum_n f'_n
  double fp_thresh = 0.0;    // 1e-14 * sum_k w_k nocc_k
  pwb::DevBuf phi, d_off, d_nocc, d_band_k, d_eps, d_pshift, d_coef, vloc, rho, wt;
  pwb::DevBuf psir;          // psi(r) cache for rows [shard_b0, shard_b1)
  int psir_b0 = -1, psir_b1 = -1;
  // chi0 workspaces
  pwb::DevBuf dvpsi, dphi, cm, cw, part, fsum, drho_part, scal;
  int shard_b0 = 0, shard_b1 = 0;
  pwb::ProjPlan shard_plan;
  pwb::CgBatch cg;           // batch over the shard rows (reused across chi0 calls)
  pwb::CgBatch cg_user;      // batch for pwb_sternheimer calls
  pwb::ProjPlan user_plan;   // pwb_project_out
  std::vector<int> user_plan_key;
};
