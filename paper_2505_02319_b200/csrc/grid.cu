// Grid/FFT plan construction and the sphere<->cube C-ABI entry points.
#include <cmath>
#include <cstring>
#include <algorithm>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "grid.cuh"

namespace pwb {

unsigned long long g_launches = 0;
bool g_pdl = getenv("PWB_NO_PDL") == nullptr;
static thread_local std::string t_err;
void set_error(const std::string& msg) { t_err = msg; }
const char* last_error() { return t_err.c_str(); }

int DevBuf::ensure(size_t need) {
  if (need <= bytes && ptr) return PWB_OK;
  release();
  if (need == 0) return PWB_OK;
  cudaError_t e = cudaMalloc(&ptr, need);
  if (e != cudaSuccess) {
    ptr = nullptr;
    bytes = 0;
    cudaGetLastError();
    return fail(PWB_ERR_NOMEM, std::string("cudaMalloc(") + std::to_string(need) +
                                   "): " + cudaGetErrorString(e));
  }
  bytes = need;
  return PWB_OK;
}

void DevBuf::release() {
  if (ptr) cudaFree(ptr);
  ptr = nullptr;
  bytes = 0;
}

static int radix_plan(int n, LinePlan& pl) {
  pl.n = n;
  pl.code = 0;
  int npass = 0;
  int m = n;
  while (m > 1) {
    int r;
    if (m % 8 == 0) r = 8;
    else if (m % 4 == 0) r = 4;
    else if (m % 2 == 0) r = 2;
    else if (m % 3 == 0) r = 3;
    else if (m % 5 == 0) r = 5;
    else return fail(PWB_ERR_UNSUPPORTED, "FFT length " + std::to_string(n) + " is not 5-smooth");
    if (npass >= kMaxPasses) return fail(PWB_ERR_UNSUPPORTED, "FFT length too large");
    pl.code |= (unsigned)r << (4 * npass);
    ++npass;
    m /= r;
  }
  return PWB_OK;
}

template <typename T>
static int upload(pwb_grid* g, const T* host, size_t count, const T** dev) {
  void* p = nullptr;
  size_t bytes = count * sizeof(T);
  if (bytes == 0) bytes = sizeof(T);
  cudaError_t e = cudaMalloc(&p, bytes);
  if (e != cudaSuccess) return fail(PWB_ERR_NOMEM, std::string("cudaMalloc: ") + cudaGetErrorString(e));
  g->owned.push_back(p);
  if (count) PWB_CUDA(cudaMemcpy(p, host, count * sizeof(T), cudaMemcpyHostToDevice));
  *dev = reinterpret_cast<const T*>(p);
  return PWB_OK;
}

static int twiddles(pwb_grid* g, int n, const double2** dev) {
  std::vector<double2> tw(n);
  for (int m = 0; m < n; ++m) {
    long double ang = -2.0L * 3.141592653589793238462643383279502884L * (long double)m / n;
    tw[m] = make_double2((double)cosl(ang), (double)sinl(ang));
  }
  return upload(g, tw.data(), (size_t)n, dev);
}

static inline int wrap(int i, int n) { return ((i % n) + n) % n; }

}  // namespace pwb

using namespace pwb;

extern "C" {

const char* pwb_last_error(void) { return pwb::last_error(); }
int pwb_version(void) { return 1; }
unsigned long long pwb_launch_count(void) { return pwb::g_launches; }

int pwb_device_count(int* count) {
  int n = 0;
  cudaError_t e = cudaGetDeviceCount(&n);
  if (e != cudaSuccess) {
    cudaGetLastError();
    n = 0;
  }
  *count = n;
  return PWB_OK;
}

int pwb_grid_set_stream(pwb_grid* g, void* stream) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  g->stream = reinterpret_cast<cudaStream_t>(stream);
  return PWB_OK;
}

int pwb_grid_create(int nx, int ny, int nz, double volume, int nk, const int* nb_per_k,
                    const int* g_int, const double* g2_sphere, const double* g2_cube,
                    pwb_grid** out) {
  if (!out) return fail(PWB_ERR_VALUE, "null output pointer");
  *out = nullptr;
  if (nx < 1 || ny < 1 || nz < 1 || nk < 1 || !(volume > 0))
    return fail(PWB_ERR_VALUE, "invalid grid dimensions");
  int ndev = 0;
  pwb_device_count(&ndev);
  if (ndev == 0) return fail(PWB_ERR_CUDA, "no CUDA device available");
  auto* g = new pwb_grid();
  std::unique_ptr<pwb_grid> guard(g);
  g->nx = nx;
  g->ny = ny;
  g->nz = nz;
  g->nyz = ny * nz;
  g->ng = nx * ny * nz;
  g->volume = volume;
  g->nk = nk;
  g->nb.assign(nb_per_k, nb_per_k + nk);
  int maxnb = 0;
  size_t tot = 0;
  for (int k = 0; k < nk; ++k) {
    if (g->nb[k] < 1) return fail(PWB_ERR_VALUE, "empty sphere");
    maxnb = std::max(maxnb, g->nb[k]);
    tot += g->nb[k];
  }
  g->nbp = ((maxnb + 63) / 64) * 64;

  int ixmin = 1 << 30, ixmax = -(1 << 30), iymin = 1 << 30, iymax = -(1 << 30);
  for (size_t s = 0; s < tot; ++s) {
    ixmin = std::min(ixmin, g_int[3 * s]);
    ixmax = std::max(ixmax, g_int[3 * s]);
    iymin = std::min(iymin, g_int[3 * s + 1]);
    iymax = std::max(iymax, g_int[3 * s + 1]);
  }
  g->ixmin = ixmin;
  g->iymin = iymin;
  g->nxa = ixmax - ixmin + 1;
  g->nya = iymax - iymin + 1;
  if (g->nxa > nx || g->nya > ny) return fail(PWB_ERR_CONFIG, "sphere does not fit the cube");

  std::vector<int> xa(g->nxa), ya(g->nya), xall(nx), yall(ny);
  for (int p = 0; p < g->nxa; ++p) xa[p] = wrap(ixmin + p, nx);
  for (int q = 0; q < g->nya; ++q) ya[q] = wrap(iymin + q, ny);
  for (int i = 0; i < nx; ++i) xall[i] = i;
  for (int i = 0; i < ny; ++i) yall[i] = i;

  g->xr_host.assign((size_t)nk * (g->nxa + 1), 0);
  std::vector<int> pp((size_t)nk * g->nbp, 0), ppp((size_t)nk * g->nbp, 0);
  std::vector<double> kin((size_t)nk * g->nbp, 0.0);
  const int nyp = (ny % 2 == 0) ? ny + 1 : ny;
  size_t off = 0;
  for (int k = 0; k < nk; ++k) {
    int* xr = &g->xr_host[(size_t)k * (g->nxa + 1)];
    std::vector<int> count(g->nxa, 0);
    int prev = -(1 << 30);
    for (int s = 0; s < g->nb[k]; ++s) {
      const int* gi = g_int + 3 * (off + s);
      if (gi[0] < prev) return fail(PWB_ERR_VALUE, "sphere is not sorted by the first index");
      prev = gi[0];
      count[gi[0] - ixmin]++;
      pp[(size_t)k * g->nbp + s] = wrap(gi[2], nz) * ny + wrap(gi[1], ny);
      ppp[(size_t)k * g->nbp + s] = wrap(gi[2], nz) * nyp + wrap(gi[1], ny);
      kin[(size_t)k * g->nbp + s] = 0.5 * g2_sphere[off + s];
    }
    xr[0] = 0;
    for (int p = 0; p < g->nxa; ++p) xr[p + 1] = xr[p] + count[p];
    off += g->nb[k];
  }
  std::vector<double> g2w((size_t)g->ng);
  for (int x = 0; x < nx; ++x)
    for (int z = 0; z < nz; ++z)
      for (int y = 0; y < ny; ++y)
        g2w[(size_t)x * g->nyz + (size_t)z * ny + y] = g2_cube[x + (size_t)nx * (y + (size_t)ny * z)];

  GridDev& d = g->dev;
  d.nx = nx;
  d.ny = ny;
  d.nz = nz;
  d.nyz = g->nyz;
  d.ng = g->ng;
  d.nxa = g->nxa;
  d.nya = g->nya;
  d.nk = nk;
  d.nbp = g->nbp;
  int T = 3072 / nx;
  if (T < 1) T = 1;
  if (T > g->nyz) T = g->nyz;
  d.tile = T;
  d.tilep = (T % 2 == 0) ? T + 1 : T;
  PWB_TRY(upload(g, xa.data(), xa.size(), &d.xa));
  PWB_TRY(upload(g, ya.data(), ya.size(), &d.ya));
  PWB_TRY(upload(g, xall.data(), xall.size(), &d.xall));
  PWB_TRY(upload(g, yall.data(), yall.size(), &d.yall));
  PWB_TRY(upload(g, g->xr_host.data(), g->xr_host.size(), &d.xr));
  PWB_TRY(upload(g, pp.data(), pp.size(), &d.pp));
  PWB_TRY(upload(g, ppp.data(), ppp.size(), &d.ppp));
  d.nyp = nyp;
  PWB_TRY(upload(g, kin.data(), kin.size(), &d.kin));
  PWB_TRY(upload(g, g2w.data(), g2w.size(), &d.g2w));
  PWB_TRY(radix_plan(nx, d.px));
  PWB_TRY(radix_plan(ny, d.py));
  PWB_TRY(radix_plan(nz, d.pz));
  PWB_TRY(twiddles(g, nx, &d.px.tw));
  PWB_TRY(twiddles(g, ny, &d.py.tw));
  PWB_TRY(twiddles(g, nz, &d.pz.tw));
  PWB_TRY(configure_kernels(g));
  *out = guard.release();
  return PWB_OK;
}

int pwb_grid_destroy(pwb_grid* g) {
  if (!g) return PWB_OK;
  cudaDeviceSynchronize();
  for (void* p : g->owned) cudaFree(p);
  delete g;
  return PWB_OK;
}

int pwb_grid_info(const pwb_grid* g, int* info) {
  if (!g || !info) return fail(PWB_ERR_VALUE, "null argument");
  info[0] = g->nx;
  info[1] = g->ny;
  info[2] = g->nz;
  info[3] = g->nk;
  info[4] = g->nbp;
  info[5] = g->nxa;
  info[6] = g->nya;
  info[7] = g->dev.tile;
  return PWB_OK;
}

int pwb_to_real(pwb_grid* g, int nband, const int* band_k, const double* psi, double* out) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  PWB_TRY(g->wbuf.ensure((size_t)nband * g->nxa * g->nyz * sizeof(double2)));
  double2* W = as<double2>(g->wbuf);
  PWB_TRY(launch_plane_inv(g, nband, band_k, reinterpret_cast<const double2*>(psi), 1.0, W));
  PWB_TRY(launch_pencil_to_cube(g, nband, W, 1.0 / std::sqrt(g->volume),
                                reinterpret_cast<double2*>(out)));
  return PWB_OK;
}

int pwb_to_fourier(pwb_grid* g, int nband, const int* band_k, const double* values, double* out) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  PWB_TRY(g->wbuf.ensure((size_t)nband * g->nxa * g->nyz * sizeof(double2)));
  double2* W = as<double2>(g->wbuf);
  PWB_TRY(launch_pencil_from_cube(g, nband, reinterpret_cast<const double2*>(values), W));
  PWB_TRY(launch_plane_fwd(g, nband, band_k, W, std::sqrt(g->volume) / g->ng, nullptr, nullptr,
                           reinterpret_cast<double2*>(out)));
  return PWB_OK;
}

int pwb_ham_apply(pwb_grid* g, int nband, const int* band_k, const double* psi,
                  const double* v_local, const double* shift, double* out) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  PWB_TRY(g->wbuf.ensure((size_t)nband * g->nxa * g->nyz * sizeof(double2)));
  double2* W = as<double2>(g->wbuf);
  const double2* p = reinterpret_cast<const double2*>(psi);
  PWB_TRY(g->vt.ensure((size_t)g->ng * sizeof(double)));
  PWB_TRY(launch_transpose_v(g, v_local, as<double>(g->vt)));
  PWB_TRY(launch_plane_inv(g, nband, band_k, p, 1.0, W));
  PWB_TRY(launch_pencil_vmul(g, nband, W, as<double>(g->vt), 1.0 / g->ng));
  PWB_TRY(launch_plane_fwd(g, nband, band_k, W, 1.0, p, shift, reinterpret_cast<double2*>(out)));
  return PWB_OK;
}

int pwb_ham_apply_host(pwb_grid* g, int nband, const int* band_k_host, const double* psi_host,
                       const double* v_local_host, const double* shift_host, double* out_host) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  const size_t rows = (size_t)nband * g->nbp * 2 * sizeof(double);
  DevBuf dpsi, dout, dv, dk, dsh;
  PWB_TRY(dpsi.ensure(rows));
  PWB_TRY(dout.ensure(rows));
  PWB_TRY(dv.ensure((size_t)g->ng * sizeof(double)));
  PWB_CUDA(cudaMemcpyAsync(dpsi.ptr, psi_host, rows, cudaMemcpyHostToDevice, g->stream));
  PWB_CUDA(cudaMemsetAsync(dout.ptr, 0, rows, g->stream));
  PWB_CUDA(cudaMemcpyAsync(dv.ptr, v_local_host, (size_t)g->ng * sizeof(double),
                           cudaMemcpyHostToDevice, g->stream));
  const int* bk = nullptr;
  const double* sh = nullptr;
  if (band_k_host) {
    PWB_TRY(dk.ensure((size_t)nband * sizeof(int)));
    PWB_CUDA(cudaMemcpyAsync(dk.ptr, band_k_host, (size_t)nband * sizeof(int),
                             cudaMemcpyHostToDevice, g->stream));
    bk = as<int>(dk);
  }
  if (shift_host) {
    PWB_TRY(dsh.ensure((size_t)nband * sizeof(double)));
    PWB_CUDA(cudaMemcpyAsync(dsh.ptr, shift_host, (size_t)nband * sizeof(double),
                             cudaMemcpyHostToDevice, g->stream));
    sh = as<double>(dsh);
  }
  PWB_TRY(pwb_ham_apply(g, nband, bk, as<double>(dpsi), as<double>(dv), sh, as<double>(dout)));
  PWB_CUDA(cudaMemcpyAsync(out_host, dout.ptr, rows, cudaMemcpyDeviceToHost, g->stream));
  PWB_CUDA(cudaStreamSynchronize(g->stream));
  return PWB_OK;
}

int pwb_cube_fft(pwb_grid* g, int nvec, const double* in, double* out, int inverse) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  PWB_TRY(g->wfull.ensure((size_t)nvec * g->ng * sizeof(double2)));
  double2* Wf = as<double2>(g->wfull);
  PWB_TRY(launch_full_from_natural(g, nvec, reinterpret_cast<const double2*>(in), nullptr,
                                   inverse ? 2 : 1, Wf));
  PWB_TRY(launch_full_plane(g, nvec, Wf, 0, 0.0, inverse));
  PWB_TRY(launch_full_to_natural(g, nvec, Wf, 0, inverse ? 1.0 / g->ng : 1.0,
                                 reinterpret_cast<double2*>(out), nullptr, nullptr, nullptr));
  return PWB_OK;
}

int pwb_kernel_apply(pwb_grid* g, int lda_x, const double* rho, const double* v, double* out) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  PWB_TRY(g->wfull.ensure((size_t)g->ng * sizeof(double2)));
  double2* Wf = as<double2>(g->wfull);
  PWB_TRY(launch_full_from_natural(g, 1, nullptr, v, 1, Wf));
  PWB_TRY(launch_full_plane(g, 1, Wf, 1, 0.0, 0));
  PWB_TRY(launch_full_to_natural(g, 1, Wf, 2, 1.0 / g->ng, nullptr, out, lda_x ? v : nullptr,
                                 lda_x ? rho : nullptr));
  return PWB_OK;
}

int pwb_kerker_apply(pwb_grid* g, double alpha, const double* v, double* out) {
  if (!g) return fail(PWB_ERR_VALUE, "null grid");
  if (!(alpha >= 0)) return fail(PWB_ERR_CONFIG, "kerker alpha must be >= 0");
  if (alpha == 0.0) {
    PWB_CUDA(cudaMemcpyAsync(out, v, (size_t)g->ng * sizeof(double), cudaMemcpyDeviceToDevice,
                             g->stream));
    return PWB_OK;
  }
  PWB_TRY(g->wfull.ensure((size_t)g->ng * sizeof(double2)));
  double2* Wf = as<double2>(g->wfull);
  PWB_TRY(launch_full_from_natural(g, 1, nullptr, v, 1, Wf));
  PWB_TRY(launch_full_plane(g, 1, Wf, 2, alpha, 0));
  PWB_TRY(launch_full_to_natural(g, 1, Wf, 2, 1.0 / g->ng, nullptr, out, nullptr, nullptr));
  return PWB_OK;
}

}  // extern "C"
