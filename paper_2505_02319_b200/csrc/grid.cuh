// Grid / FFT plan object and its device view.
//
// HBM layouts:
//   sphere rows  psi[b][nbp]             complex, lexicographic G order, zero pad
//   plane buffer W[b][p][z][y]           complex, p = active x plane (signed ix
//                                        ascending), y fastest -- the pruned
//                                        intermediate of every sphere<->cube
//                                        transform; only nxa of nx planes exist
//   natural cube u[b][z][y][x]           complex or real, x fastest (reference)
#pragma once

#include <vector>

#include "common.cuh"
#include "fft_engine.cuh"

namespace pwb {

struct GridDev {
  int nx, ny, nz, nyz, ng;
  int nxa, nya;   // active x planes / active y lines (pruned transforms)
  int nk, nbp;
  int tile, tilep;  // pencil tile (yz points per CTA) and its odd smem stride
  const int* xa;    // [nxa]   wrapped x of active plane p
  const int* ya;    // [nya]   wrapped y of active line
  const int* xall;  // [nx]    identity (full transforms)
  const int* yall;  // [ny]
  const int* xr;    // [nk][nxa+1] sphere offsets of plane p
  const int* pp;    // [nk][nbp]   in-plane index iz*ny+iy of each sphere point
  const int* ppp;   // [nk][nbp]   same in the padded smem plane: iz*nyp+iy
  int nyp;          // smem plane row stride: ny rounded up to odd (bank-conflict free)
  const double* kin;  // [nk][nbp] |G+k|^2 / 2
  const double* g2w;  // [nx][nz][ny] |G|^2 in plane layout (full cube)
  LinePlan px, py, pz;
};

struct DevBuf {
  void* ptr = nullptr;
  size_t bytes = 0;
  int ensure(size_t need);
  void release();
  ~DevBuf() { release(); }
};

template <typename T>
inline T* as(DevBuf& b) { return reinterpret_cast<T*>(b.ptr); }

}  // namespace pwb

struct pwb_grid {
  int nx, ny, nz, nyz, ng;
  double volume;
  int nk, nbp, nxa, nya, ixmin, iymin;
  std::vector<int> nb;            // per k
  std::vector<int> xr_host;       // [nk][nxa+1]
  pwb::GridDev dev;
  cudaStream_t stream = nullptr;
  // owned device tables
  std::vector<void*> owned;
  // workspaces
  pwb::DevBuf wbuf;       // plane buffer for sphere transforms
  pwb::DevBuf wfull;      // full-cube plane buffer
  pwb::DevBuf tmp_sphere; // scratch sphere rows
  pwb::DevBuf tmp_real;   // scratch real vectors
  pwb::DevBuf red;        // reduction scratch
  pwb::DevBuf scratch;    // small device scalars (GMRES)
  pwb::DevBuf mgs_part;   // per-CTA partial dots of the fused MGS step
  pwb::DevBuf mgs_bar;    // its grid-barrier counters
  pwb::DevBuf vt;         // x-major copy of a real multiplier (pencil V product)
};

namespace pwb {

// launchers (fft_kernels.cu); all asynchronous on grid->stream
// rows (optional): plane-buffer slot b reads/writes sphere row rows[b] (active-row compaction)
// nact (optional): device row count; grid rows >= *nact exit (fixed-grid graph replay)
int launch_plane_inv(pwb_grid* g, int nband, const int* band_k, const double2* psi, double scale,
                     double2* W, const int* rows = nullptr, const int* nact = nullptr);
int launch_plane_inv2(pwb_grid* g, int nband, const int* band_k, const double2* a,
                      const double2* b, double2* W);
// v must be x-major (launch_transpose_v)
int launch_pencil_vmul(pwb_grid* g, int nband, double2* W, const double* v, double vscale,
                       const int* nact = nullptr);
int launch_transpose_v(pwb_grid* g, const double* v, double* vt);
int launch_plane_fwd(pwb_grid* g, int nband, const int* band_k, const double2* W, double a,
                     const double2* psi_in, const double* shift, double2* out,
                     const int* rows = nullptr, const int* nact = nullptr);
int launch_pencil_to_cube(pwb_grid* g, int nband, const double2* W, double scale, double2* out);
// same, written x-major [band][x][yz] (the accumulation's psi(r) cache layout)
int launch_pencil_to_cube_xmajor(pwb_grid* g, int nband, const double2* W, double scale,
                                 double2* out);
int launch_pencil_from_cube(pwb_grid* g, int nband, const double2* in, double2* W);
// full-cube (all planes) helpers
// mode: 0 no x-FFT, 1 forward, 2 inverse
int launch_full_from_natural(pwb_grid* g, int nvec, const double2* in_c, const double* in_r,
                             int mode, double2* Wf);
int launch_full_plane(pwb_grid* g, int nvec, double2* Wf, int mode, double param, int inverse);
int launch_full_to_natural(pwb_grid* g, int nvec, const double2* Wf, int mode, double scale,
                           double2* out_c, double* out_r, const double* v_lda,
                           const double* rho_lda);
int configure_kernels(const pwb_grid* g);

size_t plane_smem(const pwb_grid* g);
size_t pencil_smem(const pwb_grid* g);

}  // namespace pwb
