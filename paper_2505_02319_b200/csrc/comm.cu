// Multi-GPU plumbing of the sharded chi0 (SURVEY.md 8(b) "C1", 8(e)): one
// NCCL communicator per device state and ONE all-reduce per chi0 apply, of
// the packet [drho partial | C(r) (metals) | sum w f' delta eps | failed rows |
// per-row CG iterations | failed-row residuals] written by
// pwb_chi0_finish_local (state.cu).  The reference has no counterpart: its
// only parallelism is the band thread pool of apply_chi0 (response.py:144-148).
//
// NCCL is resolved at run time (dlopen of libnccl.so.2, preferring the copy
// torch has already loaded), so the library links without it and a
// single-GPU process never touches it.
#include <dlfcn.h>
#include <nccl.h>

#include <cmath>
#include <cstring>
#include <mutex>
#include <string>

#include "state.cuh"

namespace pwb {

static thread_local double t_residual = NAN;
void set_last_residual(double r) { t_residual = r; }

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // torch's copy, if loaded
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();
      api.why = std::string("libnccl.so.2 not found: ") + (e ? e : "");
      return;
    }
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank =
        reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.error_string =
        reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.all_reduce && api.comm_destroy &&
             api.error_string;
    if (!api.ok) api.why = "libnccl.so.2 lacks a required symbol";
  });
  return api;
}

int nccl_fail(const NcclApi& api, ncclResult_t r, const char* what) {
  return fail(PWB_ERR_CUDA, std::string(what) + ": " + api.error_string(r));
}

}  // namespace

int comm_destroy(pwb_state* st) {
  if (!st->comm) return PWB_OK;
  const NcclApi& api = nccl();
  ncclComm_t c = reinterpret_cast<ncclComm_t>(st->comm);
  st->comm = nullptr;
  if (api.ok) {
    const ncclResult_t r = api.comm_destroy(c);
    if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommDestroy");
  }
  return PWB_OK;
}

}  // namespace pwb

pwb_state::~pwb_state() {
  (void)pwb::comm_destroy(this);
  if (h_tail) cudaFreeHost(h_tail);
}

using namespace pwb;

extern "C" {

double pwb_last_residual(void) { return t_residual; }

int pwb_comm_unique_id(void* id_out) {
  if (!id_out) return fail(PWB_ERR_VALUE, "null argument");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(PWB_ERR_UNSUPPORTED, api.why);
  ncclUniqueId id;
  const ncclResult_t r = api.get_unique_id(&id);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclGetUniqueId");
  memcpy(id_out, &id, sizeof(id));
  return PWB_OK;
}

int pwb_comm_init(pwb_state* st, const void* id, int rank, int nranks) {
  if (!st || !id) return fail(PWB_ERR_VALUE, "null argument");
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(PWB_ERR_VALUE, "bad rank / nranks");
  const NcclApi& api = nccl();
  if (!api.ok) return fail(PWB_ERR_UNSUPPORTED, api.why);
  PWB_TRY(comm_destroy(st));
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof(uid));
  ncclComm_t c = nullptr;
  const ncclResult_t r = api.comm_init_rank(&c, nranks, uid, rank);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclCommInitRank");
  st->comm = c;
  return PWB_OK;
}

int pwb_comm_destroy(pwb_state* st) {
  if (!st) return fail(PWB_ERR_VALUE, "null state");
  return comm_destroy(st);
}

int pwb_allreduce(pwb_state* st, double* buf, long long n) {
  if (!st || (!buf && n > 0)) return fail(PWB_ERR_VALUE, "null argument");
  if (!st->comm) return fail(PWB_ERR_CONFIG, "no communicator: call pwb_comm_init first");
  if (n <= 0) return PWB_OK;
  const NcclApi& api = nccl();
  const ncclResult_t r = api.all_reduce(buf, buf, (size_t)n, ncclFloat64, ncclSum,
                                        reinterpret_cast<ncclComm_t>(st->comm), st->g->stream);
  if (r != ncclSuccess) return nccl_fail(api, r, "ncclAllReduce");
  return PWB_OK;
}

}  // extern "C"
