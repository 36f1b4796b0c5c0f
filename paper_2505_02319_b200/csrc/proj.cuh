// Projector GEMM plans (see proj.cu).
#pragma once

#include <algorithm>
#include <vector>

#include "grid.cuh"

namespace pwb {

constexpr int kProjTileRows = 16;   // rows per projector tile (<= 2 DMMA n-fragments)
constexpr int kProjChunk = 64;      // sphere coefficients per pipeline chunk
constexpr int kProjRowStride = kProjChunk + 4;   // padded smem / chunk-major row (double2)
// wide tiles (projw.cu): up to 72 rows of one k block against all its <= 72 orbitals
constexpr int kProjWideRows = 72;
constexpr int kProjWideOcc = 72;
constexpr int kProjWideChunk = 32;

struct ProjTile {
  int row0;   // first row of X in this tile
  int nrows;  // <= kProjTileRows, all in k block `k`
  int k;
};

struct ProjArgs {
  const double2* phi;   // state orbital rows [nband][nbp]
  const int* off;       // [nk] first orbital row of block k
  const int* nocc;      // [nk]
  const ProjTile* tiles;
  int nbp;
  int ldc;              // leading dim of C / partials (max nocc)
  int nrows_total;
  const int* rows;      // optional: compact row i -> X row rows[i] (active-row compaction)
  const int* ntiles;    // optional device tile count: CTAs with blockIdx.x >= *ntiles exit
  // chunk-major copy of phi: block k, chunk c, orbital m at
  // phic + phic_off[k] + (c * nocc[k] + m) * kProjRowStride (pads zero), so the
  // orbitals of one chunk are ONE contiguous TMA bulk copy
  const double2* phic;
  const int* phic_off;  // [nk], in double2
  // the same for the wide-tile kernels (projw.cu): coef copy with narrow chunks,
  // apply copy with 32-coefficient chunks (strides chosen per access pattern)
  const double2* phiw;
  const int* phiw_off;
  const double2* phiwa;   // the apply kernel's copy (32-wide chunks, stride 38)
  const int* phiwa_off;
};

// Build the chunk-major copy of the orbital rows phi [nband][nbp] (k blocks at
// off_host[k], nocc_host[k] rows each): allocates phic, writes [off | nocc |
// phic_off] (3 nk ints) to d_phic_off -- ProjArgs::phic_off is its base + 2 nk --
// and runs the copy on `st` (synchronised before returning).
int proj_chunked(const double2* phi, int nbp, const std::vector<int>& off_host,
                 const std::vector<int>& nocc_host, DevBuf& phic, DevBuf& d_phic_off,
                 cudaStream_t st);

struct ProjPlan {
  std::vector<ProjTile> tiles;
  DevBuf dtiles;
  DevBuf counters;   // split-K arrival counters (self-resetting)
  ProjTile* h_stage = nullptr;   // pinned staging for async tile uploads
  size_t h_cap = 0;
  int nrows = 0, mtiles = 0, nsplit = 1, split_len = 0;
  int max_tiles = 0;   // > 0: tiles are produced on the device (capacity plan)
  // wide tiles (projw.cu): host list (host plans) or device capacity (wmax > 0)
  std::vector<ProjTile> wtiles;
  DevBuf dwtiles, wcounters;
  int wmax = 0;
  ~ProjPlan() {
    if (h_stage) cudaFreeHost(h_stage);
  }
};

inline int plan_tiles(const ProjPlan& pl) {
  return pl.max_tiles > 0 ? pl.max_tiles : (int)pl.tiles.size();
}

// capacity plan whose tile list (<= max_tiles entries, <= wide_tiles wide ones) is
// written on the device; launches cover the capacity and CTAs beyond the device
// count ProjArgs::ntiles exit
int proj_plan_device(ProjPlan& pl, int max_tiles, int maxocc, int nbp, int wide_tiles = 0);
inline int plan_wide_tiles(const ProjPlan& pl) {
  return pl.wmax > 0 ? pl.wmax : (int)pl.wtiles.size();
}

// build the tile list for rows with k blocks row_k; uploads synchronously, or
// asynchronously on `st` when st != nullptr (staging buffer reused: the caller
// must not rebuild the plan before that stream has passed the upload)
int proj_plan(ProjPlan& pl, const std::vector<int>& row_k, const std::vector<int>& nocc, int nbp,
              cudaStream_t st = nullptr, bool async = false);
// scratch (complex elements) needed by proj_coeffs for this plan / any plan of <= nrows rows
size_t proj_part_elems(const ProjPlan& pl);
// C = Phi^H X   (part: nsplit * nrows * ldc scratch)
int proj_coeffs(const ProjPlan& pl, ProjArgs a, const double2* X, double2* part, double2* C,
                cudaStream_t st);
// Y = ca X + cb Phi C  (rows with active[row % band_mod] == 0 untouched; active may be NULL)
int proj_apply(const ProjPlan& pl, ProjArgs a, const double2* C, const double2* Xin, double2* Y,
               double ca, double cb, const int* active, int band_mod, cudaStream_t st);

// Fused single-launch Q X for a few tiles of one orbital block (N_occ <= 40):
// every split's chunks stay in smem from the partial C to the update.
// flags: one generation counter per tile (persistent, zero-initialised).
bool proj_small_fits(int ntiles, int nbp, int maxocc);
int proj_small(const ProjPlan& pl, ProjArgs a, double2* X, const int* active, int band_mod,
               double2* part, double2* C, unsigned* flags, cudaStream_t st);

// ---- wide-tile projector (projw.cu) ----------------------------------------------
bool projw_enabled();
// wide tiles (<= kProjWideRows rows of one k block) over rows with k blocks row_k
int projw_tiles(const std::vector<int>& row_k, std::vector<ProjTile>& out);
size_t projw_part_elems(int max_tiles);
// C = Phi^H X over `cap` tiles (device count a.ntiles when set, else nt_host)
// (x_rows: rows allocated in X, bound of the TMA tensor map; <= 0: per-row copies only)
int projw_coeffs(const ProjTile* dtiles, int nt_host, int cap, ProjArgs a, const double2* X,
                 double2* part, double2* C, unsigned* counters, cudaStream_t st,
                 long long x_rows = 0);
// Y = ca X + cb Phi C
int projw_apply(const ProjTile* dtiles, int nt_host, int cap, ProjArgs a, const double2* C,
                const double2* Xin, double2* Y, double ca, double cb, const int* active,
                int band_mod, cudaStream_t st);
int projw_chunked(const double2* phi, int nbp, const std::vector<int>& off_host,
                  const std::vector<int>& nocc_host, DevBuf& phiw, DevBuf& d_meta,
                  DevBuf& phiwa, DevBuf& d_meta_a, cudaStream_t st);

}  // namespace pwb
