// pb200 — native NCCL allreduce for the sharded sweep.
//
// The dictionary step of a sharded sweep exchanges the 48·P moment sums of
// every 8-atom block (K/8 small allreduces per sweep) plus the epoch
// statistics.  Routing each through a host callback costs tens of µs of host
// work per exchange; here the exchange is an `ncclAllReduce` enqueued on the
// epoch's own stream (stream-ordered: no host synchronisation between the
// pass kernel, the allreduce and the atom-draw kernel).  NCCL is loaded with
// dlopen — the process's already-loaded libnccl.so.2 (e.g. the one PyTorch
// brought) is reused — so the library has no link-time NCCL dependency.
// `pb_nccl_allreduce` has the pb_allreduce_fn signature: a caller passes its
// address as pb_epoch_desc.allreduce with the communicator as the context.
#include <dlfcn.h>

#include <mutex>

#include "../../include/pb200.h"
#include "pb_common.cuh"

namespace {

typedef struct ncclComm* nccl_comm_t;
typedef struct {
  char internal[128];
} nccl_unique_id_t;

typedef int (*fn_get_unique_id)(nccl_unique_id_t*);
typedef int (*fn_comm_init_rank)(nccl_comm_t*, int, nccl_unique_id_t, int);
typedef int (*fn_comm_destroy)(nccl_comm_t);
typedef int (*fn_all_reduce)(const void*, void*, size_t, int, int, nccl_comm_t, cudaStream_t);
typedef const char* (*fn_error_string)(int);

struct NcclApi {
  void* handle = nullptr;
  fn_get_unique_id get_unique_id = nullptr;
  fn_comm_init_rank comm_init_rank = nullptr;
  fn_comm_destroy comm_destroy = nullptr;
  fn_all_reduce all_reduce = nullptr;
  fn_error_string error_string = nullptr;
};

std::mutex g_mu;
NcclApi g_api;

bool load_nccl() {
  std::lock_guard<std::mutex> lk(g_mu);
  if (g_api.handle) return true;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);   // the copy already in the process, if any
  if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_LOCAL);
  if (!h) {
    pb::set_error("NCCL not available: %s", dlerror());
    return false;
  }
  g_api.get_unique_id = (fn_get_unique_id)dlsym(h, "ncclGetUniqueId");
  g_api.comm_init_rank = (fn_comm_init_rank)dlsym(h, "ncclCommInitRank");
  g_api.comm_destroy = (fn_comm_destroy)dlsym(h, "ncclCommDestroy");
  g_api.all_reduce = (fn_all_reduce)dlsym(h, "ncclAllReduce");
  g_api.error_string = (fn_error_string)dlsym(h, "ncclGetErrorString");
  if (!g_api.get_unique_id || !g_api.comm_init_rank || !g_api.comm_destroy || !g_api.all_reduce) {
    pb::set_error("libnccl.so.2 lacks the expected symbols");
    return false;
  }
  g_api.handle = h;
  return true;
}

int nccl_fail(const char* what, int r) {
  pb::set_error("%s failed: %s", what, g_api.error_string ? g_api.error_string(r) : "nccl error");
  return PB_ECUDA;
}

}  // namespace

extern "C" {

int pb_nccl_unique_id(uint8_t* id_out) {
  if (!id_out) { pb::set_error("null argument"); return PB_EVALUE; }
  if (!load_nccl()) return PB_EUNSUPPORTED;
  nccl_unique_id_t id;
  const int r = g_api.get_unique_id(&id);
  if (r) return nccl_fail("ncclGetUniqueId", r);
  memcpy(id_out, id.internal, 128);
  return PB_OK;
}

int pb_nccl_comm_create(const uint8_t* id, int32_t world, int32_t rank, void** comm_out) {
  if (!id || !comm_out || world < 1 || rank < 0 || rank >= world) { pb::set_error("bad argument"); return PB_EVALUE; }
  if (!load_nccl()) return PB_EUNSUPPORTED;
  nccl_unique_id_t uid;
  memcpy(uid.internal, id, 128);
  nccl_comm_t comm = nullptr;
  const int r = g_api.comm_init_rank(&comm, world, uid, rank);
  if (r) return nccl_fail("ncclCommInitRank", r);
  *comm_out = comm;
  return PB_OK;
}

int pb_nccl_comm_destroy(void* comm) {
  if (!comm) return PB_OK;
  if (!load_nccl()) return PB_EUNSUPPORTED;
  const int r = g_api.comm_destroy((nccl_comm_t)comm);
  return r ? nccl_fail("ncclCommDestroy", r) : PB_OK;
}

// pb_allreduce_fn: in-place sum, dtype 0 = f64, 1 = i32 (the epoch's exchanges)
int pb_nccl_allreduce(void* comm, void* device_buf, int64_t count, int32_t dtype, void* stream) {
  if (!comm || !device_buf || count < 0) { pb::set_error("bad argument"); return PB_EVALUE; }
  if (!g_api.all_reduce && !load_nccl()) return PB_EUNSUPPORTED;
  const int nccl_dtype = dtype == 0 ? 8 /* ncclFloat64 */ : dtype == 1 ? 2 /* ncclInt32 */ : -1;
  if (nccl_dtype < 0) { pb::set_error("unsupported allreduce dtype %d", dtype); return PB_EVALUE; }
  const int r = g_api.all_reduce(device_buf, device_buf, (size_t)count, nccl_dtype, 0 /* ncclSum */,
                                 (nccl_comm_t)comm, (cudaStream_t)stream);
  return r ? nccl_fail("ncclAllReduce", r) : PB_OK;
}

}  // extern "C"
