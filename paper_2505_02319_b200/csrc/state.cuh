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

// Device-side iteration control written by the compaction kernel each CG
// iteration: counts, the active-row lists and the projector tile lists.
struct IterCtl {
  int* hdr;        // [0] na, [1] tiles A, [2] tiles B, [3] active count, [4] fail flag
  int* rows;       // [n]   active rows, ascending
  int* rows2;      // [2n]  stacked (x; r) buffer rows, k-interleaved: per k its rows, then its rows + n
  ProjTile* ta;    // tiles over rows
  ProjTile* tb;    // tiles over rows2
  ProjTile* wa;    // wide tiles (projw.cu) over rows, or null
  ProjTile* wb;    // wide tiles over rows2
  int wide_min;    // average live rows per wide tile from which the wide path runs
};
int projw_min_rows();
// ints of IterCtl::hdr: [0] na, [1] tiles A, [2] tiles B, [3] rows still iterating,
// [4] failure flag, [5] loop count, [6] loop cap, [8] wide tiles A, [9] wide tiles B
constexpr int kHdrInts = 16;

struct CgBatch {
  int nrows = 0;
  std::vector<int> bands;   // global band of each row
  ProjPlan plan1;           // rows [0, n) (init / RHS)
  ProjPlan pa, pb;          // device-tile plans (compacted rows / stacked rows)
  DevBuf xr, z, p, ap, rhs;
  DevBuf scal;              // CgScalars storage
  DevBuf part, cmat;        // GEMM scratch
  DevBuf ctl_buf;           // IterCtl storage
  IterCtl ctl;
  CgScalars s;
  int* h_hdr = nullptr;     // pinned copy of ctl.hdr
  int* h_its = nullptr;     // pinned per-row iteration counts / residuals (readback)
  double* h_res = nullptr;
  int h_rows = 0;
  bool loop_ran = false;    // the last cg_solve ran the device-loop graph
  int max_tiles = 0;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t exec = nullptr;
  cudaStream_t graph_stream = nullptr;
  void* graph_w = nullptr;  // plane buffer captured in the graph
  void* graph_part = nullptr;   // GEMM scratch captured in the graph
  void* graph_cmat = nullptr;
  bool loop_graph = false;  // graph = WHILE conditional node around one iteration
  int prof_rows = 0;        // active rows of the running iteration (profiler units)
  ~CgBatch();
};

constexpr int kMaxK = 128;  // k blocks handled by the device-side compaction

// batched PCG (cg.cu)
ProjArgs proj_args(pwb_state* st);
int project_rows(pwb_state* st, const ProjPlan& pl, double2* X, const int* active, int band_mod,
                 const int* rows, double2* part, double2* cmat, cudaStream_t s,
                 const int* ntiles = nullptr, int mult = 1, const int* wntiles = nullptr);
// C = Phi^H X / Y = ca X + cb Phi C through the wide-tile kernels when the state
// and plan allow them (device tile counts: a.ntiles for 16-row tiles, wntiles for
// wide ones), else the 16-row kernels of proj.cu
int proj_coeffs_any(pwb_state* st, const ProjPlan& pl, ProjArgs a, const double2* X,
                    double2* part, double2* C, cudaStream_t s, const int* wntiles = nullptr,
                    long long x_rows = 0);
int proj_apply_any(pwb_state* st, const ProjPlan& pl, ProjArgs a, const double2* C,
                   const double2* Xin, double2* Y, double ca, double cb, const int* active,
                   int band_mod, cudaStream_t s, const int* wntiles = nullptr);
int cg_setup(pwb_state* st, CgBatch& cg, const std::vector<int>& bands);
// defer: enqueue the result readback and return without synchronising; the
// caller synchronises the stream (after queueing more work) and calls cg_check
int cg_solve(pwb_state* st, CgBatch& cg, const std::vector<double>& tol, int max_iter,
             int* iters_host, double* res_host, bool defer = false);
int cg_check(CgBatch& cg, const std::vector<double>& tol, int* iters_host, double* res_host);

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
  pwb::DevBuf vloct;         // x-major V_local for the fused pencil multiply
  pwb::DevBuf phic, phic_meta;   // chunk-major orbitals for the projector (proj.cuh)
  pwb::DevBuf phiw, phiw_meta, phiwa, phiwa_meta;   // chunk-major orbitals of projw.cu
  bool wide_ok = false;          // every k block has <= kProjWideOcc orbitals
  pwb::DevBuf psir;          // psi(r) cache for rows [shard_b0, shard_b1)
  int psir_b0 = -1, psir_b1 = -1;
  // chi0 workspaces
  pwb::DevBuf dvpsi, dphi, cm, cw, part, fsum, drho_part, scal;
  int shard_b0 = 0, shard_b1 = 0;
  pwb::ProjPlan shard_plan;
  pwb::CgBatch cg;           // batch over the shard rows (reused across chi0 calls)
  pwb::CgBatch cg_user;      // batch for pwb_sternheimer calls
  pwb::ProjPlan user_plan;   // pwb_project_out
  pwb::DevBuf user_part, user_cmat;   // pwb_project_out scratch (never cg_user's: its graph
                                      // captured cg_user.part / cmat pointers)
  pwb::DevBuf small_flags;   // per-tile generation flags of the fused small projector
  std::vector<int> user_plan_key;
  // sharded chi0 (comm.cu): NCCL communicator, cached C(r) of the shard rows,
  // pinned readback of the reduced packet tail
  void* comm = nullptr;
  pwb::DevBuf fermi_c;
  int fermi_b0 = -1, fermi_b1 = -1;
  double* h_tail = nullptr;
  size_t h_tail_n = 0;
  ~pwb_state();
};

extern "C" int pwb_allreduce(pwb_state* st, double* buf, long long n);
namespace pwb {
void set_last_residual(double r);
int comm_destroy(pwb_state* st);
}
