/*
 * pwb200.h -- C-ABI of libpwb200.so, the B200-native (sm_100a) chi0 /
 * Sternheimer hot path for the pwdyson Dyson solver (arXiv 2505.02319).
 *
 * The reference package is pure Python and has no FFI of its own (SURVEY.md
 * section 8b); these entry points are what its operator API for the path
 * would bind.  Each declaration cites the reference function it replaces
 * (paths relative to the reference's pkg/src/pwdyson/).  INTEGRATION.md shows
 * the ctypes binding a pwdyson maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only; complex128 = interleaved (re, im) double
 *    pairs.  Functions ending in _host take HOST pointers and do the
 *    host<->device copies themselves; all other array arguments are DEVICE
 *    pointers.
 *  - Sphere vectors ("bands") are rows of length nbp (padded sphere size,
 *    pwb_grid_info) in the lexicographic G order of the reference
 *    (pwbasis.py:123-132); pad entries are zero.  Real-space vectors are
 *    flat x-fastest, index = ix + Nx*(iy + Ny*iz) (pwbasis.py:18-19).
 *  - Every function returns 0 on success or a PWB_ERR_* code; the message
 *    is available from pwb_last_error() (thread-local).  No C++ exceptions
 *    cross the ABI.  Codes map to the reference exceptions: VALUE ->
 *    ValueError, CONFIG -> ConfigurationError, NONCONV -> NonConvergenceError
 *    (errors.py:8-22), CUDA/NOMEM/UNSUPPORTED -> PwdysonError.
 *  - Results are deterministic run-to-run (fixed-order reductions, no
 *    floating-point atomics).
 */
#ifndef PWB200_H
#define PWB200_H

#ifdef __cplusplus
extern "C" {
#endif

enum {
  PWB_OK = 0,
  PWB_ERR_VALUE = 1,
  PWB_ERR_CONFIG = 2,
  PWB_ERR_NONCONV = 3,
  PWB_ERR_CUDA = 4,
  PWB_ERR_UNSUPPORTED = 5,
  PWB_ERR_NOMEM = 6
};

typedef struct pwb_grid pwb_grid;   /* sphere/cube tables + FFT plans (one or more k) */
typedef struct pwb_state pwb_state; /* ground state resident on the device */

/* ---- library ------------------------------------------------------------- */
const char* pwb_last_error(void);
int pwb_version(void);
/* number of CUDA kernels this library has launched (for launch accounting) */
unsigned long long pwb_launch_count(void);
/* CUDA device count visible to the library (0 when no GPU) */
int pwb_device_count(int* count);
/* stream used by subsequent calls on this grid/state (cudaStream_t, NULL = legacy) */
int pwb_grid_set_stream(pwb_grid* grid, void* stream);

/* live kernel timing (CUDA events on the launching stream) per category:
 * 0 H apply in CG, 1 projector GEMMs, 2 CG reductions/updates, 3 chi0 RHS,
 * 4 drho accumulation; arrays of 8.  units = rows (bands) processed.        */
int pwb_profile_enable(int on);
int pwb_profile_reset(void);
int pwb_profile_read(double* ms, long long* count, long long* units);
/* the same split as a histogram over floor(log2(live rows)): ms[cat * 16 + bucket] */
int pwb_profile_hist(double* ms, long long* count);

/* ---- grid / FFT plan:  FourierGrids (pwbasis.py:95-224) --------------------
 * nk k-point spheres sharing one (nx,ny,nz) cube.  g_int: concatenation over
 * k of (nb_k, 3) int32 integer coordinates (lexicographically sorted);
 * g2_sphere: concatenation of |G+k|^2; g2_cube: |G|^2 on the cube, x fastest
 * (pwbasis.py:152-159).  volume: cell volume |Omega|.                       */
int pwb_grid_create(int nx, int ny, int nz, double volume, int nk, const int* nb_per_k,
                    const int* g_int, const double* g2_sphere, const double* g2_cube,
                    pwb_grid** out);
int pwb_grid_destroy(pwb_grid* grid);
/* info[0..7] = nx, ny, nz, nk, nbp, nxa (active x planes), nya (active y lines), tile */
int pwb_grid_info(const pwb_grid* grid, int* info);

/* to_real_many (pwbasis.py:200-207): nband sphere rows -> complex grid values
 * out[b][n_g] = n_g/sqrt(Omega) * ifftn(Z psi_b).  band_k: device int per row
 * (NULL = all k=0).                                                          */
int pwb_to_real(pwb_grid* grid, int nband, const int* band_k, const double* psi, double* out);
/* to_fourier_many (pwbasis.py:209-214): complex grid values -> sphere rows    */
int pwb_to_fourier(pwb_grid* grid, int nband, const int* band_k, const double* values,
                   double* out);
/* apply_hamiltonian (groundstate.py:211-219), batched over rows:
 *   out_b = (|G+k|^2/2 - shift_b) psi_b + to_fourier(v_local * to_real(psi_b))
 * shift: device double per row or NULL.  Does not touch any counter; the
 * Python layer adds the count (groundstate.py:218).                         */
int pwb_ham_apply(pwb_grid* grid, int nband, const int* band_k, const double* psi,
                  const double* v_local, const double* shift, double* out);
int pwb_ham_apply_host(pwb_grid* grid, int nband, const int* band_k_host, const double* psi_host,
                       const double* v_local_host, const double* shift_host, double* out_host);
/* cube_fft / cube_ifft (pwbasis.py:218-224) of complex vectors, unnormalised
 * forward (sign -1) or 1/n_g inverse.                                         */
int pwb_cube_fft(pwb_grid* grid, int nvec, const double* in, double* out, int inverse);
/* apply_kernel (kernels.py:40-57): K v = ifft(4pi/|G|^2 fft v).real (G=0 -> 0)
 * minus (1/3)(3/pi)^(1/3) max(rho,1e-10)^(-2/3) v when lda_x != 0.           */
int pwb_kernel_apply(pwb_grid* grid, int lda_x, const double* rho, const double* v, double* out);
/* apply_kerker (kernels.py:60-70): T v = ifft(|G|^2/(|G|^2+alpha^2) fft v).real,
 * D(0) = 1; alpha == 0 -> copy.                                               */
int pwb_kerker_apply(pwb_grid* grid, double alpha, const double* v, double* out);

/* ---- ground state on device: GroundState (groundstate.py:280-326) ---------
 * Per k block: nocc_k occupied orbitals (rows of nb_k complex, i.e. the
 * transpose of phi[:, :n_occ]), eps/occ/fprime per occupied band, weight w_k.
 * v_local / rho: n_g, x fastest.  Copies everything (host pointers).          */
int pwb_state_create(pwb_grid* grid, const int* nocc_per_k, const double* kweight,
                     const double* phi, const double* eps, const double* occ,
                     const double* fprime, const double* v_local, const double* rho,
                     pwb_state** out);
int pwb_state_destroy(pwb_state* st);
/* total occupied (k, n) pairs */
int pwb_state_nbands(const pwb_state* st, int* nbands);

/* project_out_occupied (sternheimer.py:28-30) on ncol rows of k block k:
 * x <- x - Phi_k (Phi_k^H x), in place (device rows of nbp).                 */
int pwb_project_out(pwb_state* st, int k, int ncol, double* x);

/* solve_sternheimer (sternheimer.py:33-98), batched: one projected PCG per
 * rhs row.  band[i] = global occupied-band index ((k, n) pair, block order)
 * defining Phi_k, eps_n and the preconditioner shift max(eps_n, 0.1).
 * tol[i] absolute l2 tolerance; max_iter <= 0 means 10*nb_k.  Outputs:
 * x (device rows), iters[i], res[i] (host).  Returns PWB_ERR_NONCONV if any
 * row exceeds max_iter (its residual is in res[i], iters[i] = -1).         */
int pwb_sternheimer(pwb_state* st, int nrhs, const int* band_host, const double* rhs,
                    const double* tol_host, int max_iter, double* x, int* iters_host,
                    double* res_host);

/* apply_chi0 (response.py:110-161) for the whole (k, n) batch:
 * drho = sum_k w_k sum_n [2 f_n Re(conj psi_n dphi_n) + df_n |psi_n|^2],
 * with the RHS, delta eps, the global delta eps_F, the occupied pair term
 * and one Sternheimer solve per (k, n).  dv, drho: device n_g doubles;
 * tol: host, one per (k, n); iters: host out, one per (k, n).               */
int pwb_chi0(pwb_state* st, const double* dv, const double* tol_host, double* drho,
             int* iters_host);
int pwb_chi0_host(pwb_state* st, const double* dv_host, const double* tol_host,
                  double* drho_host, int* iters_host);
/* Two-phase form for sharded (multi-GPU) use: each rank owns the band range
 * [b0, b1) of the global (k, n) list.  phase 1 computes the RHS and writes
 * fsum[0] = sum w_k f'_n delta eps_n over its bands (device double), which
 * the caller all-reduces; phase 2 finishes with the reduced fsum and the
 * host-known sum of w_k f'_n, leaving the partial drho for the caller's
 * all-reduce.                                                                */
int pwb_chi0_begin(pwb_state* st, int b0, int b1, const double* dv, double* fsum);
int pwb_chi0_finish(pwb_state* st, const double* fsum, const double* tol_host, double* drho,
                    int* iters_host);

/* ---- sharded chi0 with ONE all-reduce per apply --
 * The reference's only parallelism is the band thread pool of apply_chi0
 * (response.py:144-148); these entry points split the (k, n) list over ranks
 * instead.  After pwb_chi0_begin(b0, b1) a rank calls pwb_chi0_finish_local,
 * which runs its Sternheimer solves and accumulation with delta eps_F = 0 and
 * writes a packet of pwb_chi0_packet_size doubles (device):
 *   [drho partial (n_g) | C(r) = sum w f' |psi|^2 (n_g, metals only) |
 *    sum w f' delta eps | failed rows | CG iterations per global row (nband) |
 *    residual of each failed row, else 0 (nband)].
 * The packets are summed over ranks (pwb_allreduce: ncclAllReduce on the
 * state's stream through the communicator of pwb_comm_init, or any other
 * sum); pwb_chi0_reduce_apply then forms drho = sum - delta eps_F C(r) with
 * the global delta eps_F (response.py:131-136, summed over k) and returns the
 * iteration counts of ALL rows, failing with PWB_ERR_NONCONV on every rank if
 * any rank's row failed (residual_host = the first failed row's residual).
 * pwb_chi0_finish_sharded = local + pwb_allreduce + reduce_apply.            */
int pwb_chi0_packet_size(pwb_state* st, long long* n);
int pwb_chi0_finish_local(pwb_state* st, const double* fsum, const double* tol_host,
                          double* packet);
int pwb_chi0_reduce_apply(pwb_state* st, const double* packet, double* drho, int* iters_host,
                          double* residual_host);
int pwb_chi0_finish_sharded(pwb_state* st, const double* fsum, const double* tol_host,
                            double* packet, double* drho, int* iters_host, double* residual_host);
/* NCCL communicator of a state (NCCL resolved at run time, libnccl.so.2):
 * rank 0 calls pwb_comm_unique_id (128-byte ncclUniqueId), the caller
 * broadcasts it, every rank calls pwb_comm_init with it.                     */
int pwb_comm_unique_id(void* id_out);
int pwb_comm_init(pwb_state* st, const void* id, int rank, int nranks);
int pwb_comm_destroy(pwb_state* st);
/* in-place sum all-reduce of n device doubles on the state's stream          */
int pwb_allreduce(pwb_state* st, double* buf, long long n);
/* residual carried by the last PWB_ERR_NONCONV of this thread (NaN if none)  */
double pwb_last_residual(void);

/* orbital_row_norm (response.py:190-199): max_r sqrt(sum_n |psi_n(r)|^2)
 * (real part only when real_part != 0) over k block k.                       */
int pwb_row_norm(pwb_state* st, int k, int real_part, double* out_host);
/* same for arbitrary device sphere rows (band_k may be NULL)                 */
int pwb_row_norm_rows(pwb_grid* grid, int nrows, const int* band_k, const double* rows,
                      int real_part, double* out_host);

/* pieces of apply_chi0 for one dv (all bands): diag_host[2b], [2b+1] = Re, Im
 * of <phi_b, dv phi_b> (delta_eigen_occupations, response.py:45-71); if dphi
 * is non-NULL it receives Phi (W o M) as device rows (delta_phi_occupied,
 * response.py:101-107).                                                      */
int pwb_chi0_parts(pwb_state* st, const double* dv, double* diag_host, double* dphi);

/* project_out_occupied (sternheimer.py:28-30) for an arbitrary block: phi =
 * nocc device rows of length nb (orthonormal), x = ncol device rows, in place.
 * Asynchronous on the legacy default stream.                                  */
int pwb_project_generic(int nb, int nocc, const double* phi, int ncol, double* x);
/* same with host buffers (phi: nocc rows of nb complex, x: ncol rows, in place) */
int pwb_project_host(int nb, int nocc, const double* phi_host, int ncol, double* x_host);

/* ---- dense vector helpers for the device-resident inexact GMRES ----------
 * (igmres.py:86-114): deterministic reductions, scalars stay on device.      */
int pwb_vec_dot(pwb_grid* grid, int n, const double* x, const double* y, double* out_dev);
/* out <- a x + b y (y may be NULL: out <- a x); products and sum rounded
 * separately, i.e. numpy's `a * x + b * y` (v - |Kv| chi0, response.py:187;
 * b - E x0, igmres.py:233)                                                   */
int pwb_vec_axpby(pwb_grid* grid, long long n, double a, const double* x, double b,
                  const double* y, double* out);
/* out <- x / d (numpy's `x / d`: Kv/|Kv|, response.py:181; r0/beta, igmres.py:64) */
int pwb_vec_div(pwb_grid* grid, long long n, const double* x, double d, double* out);
/* y <- y + a x  (a host scalar) */
int pwb_vec_axpy(pwb_grid* grid, int n, double a, const double* x, double* y);
/* Arnoldi MGS step with one re-orthogonalisation pass (igmres.py:86-103):
 * V: (i+2) vectors of length n (row i+1 receives the new basis vector),
 * w: input vector (overwritten), hcol_host: i+2 entries out.               */
int pwb_arnoldi_mgs(pwb_grid* grid, int n, int i, double* basis, double* w, double* hcol_host);
/* x <- x0 + sum_j y_j V_j  (igmres.py:110-114); y host, m entries          */
int pwb_vec_combine(pwb_grid* grid, int n, int m, const double* basis, const double* y_host,
                    const double* x0, double* x);

#ifdef __cplusplus
}
#endif

#endif /* PWB200_H */
