// tm_comm.cu -- the multi-GPU exchange of the seed-partitioned path
// (SURVEY.md 8(b)/8(e)): one NCCL communicator per rank (one process per GPU),
// created from a unique id the host broadcasts, and the all-gather the ranks
// run on their device streams (NVLink / NVSwitch on one box).
//
// The library does not link NCCL: it binds the handful of entry points it
// needs from the process's libnccl.so.2 at run time (dlopen; PyTorch's copy
// when torch is loaded, else the system one), so a single-GPU user never
// needs NCCL installed.
#include <dlfcn.h>
#include <nccl.h>

#include <cstdio>
#include <cstring>
#include <mutex>
#include <string>

#include "../../include/termesh_b200.h"

namespace {

struct NcclApi {
  bool ok = false;
  std::string err;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*get_error_string)(ncclResult_t) = nullptr;
};

NcclApi& api() {
  static NcclApi a;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      a.err = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    a.all_gather = reinterpret_cast<decltype(a.all_gather)>(dlsym(h, "ncclAllGather"));
    a.get_error_string = reinterpret_cast<decltype(a.get_error_string)>(dlsym(h, "ncclGetErrorString"));
    a.ok = a.get_unique_id && a.comm_init_rank && a.comm_destroy && a.all_gather && a.get_error_string;
    if (!a.ok) a.err = "libnccl.so.2 lacks an entry point";
  });
  return a;
}

thread_local std::string g_comm_err;

int comm_fail(const char* what, ncclResult_t r) {
  char b[256];
  snprintf(b, sizeof b, "%s: %s", what, api().get_error_string ? api().get_error_string(r) : "nccl error");
  g_comm_err = b;
  return TM_ERR_CUDA;
}

}  // namespace

struct tm_comm {
  ncclComm_t comm = nullptr;
  int rank = 0, world = 1, device = 0;
};

extern "C" {

const char* tm_comm_last_error(void) { return g_comm_err.c_str(); }

int tm_comm_unique_id(void* id_out) {
  if (!id_out) return TM_ERR_ARGUMENT;
  NcclApi& a = api();
  if (!a.ok) {
    g_comm_err = a.err;
    return TM_ERR_CUDA;
  }
  ncclUniqueId id;
  ncclResult_t r = a.get_unique_id(&id);
  if (r != ncclSuccess) return comm_fail("ncclGetUniqueId", r);
  memcpy(id_out, &id, sizeof id);
  return TM_OK;
}

int tm_comm_id_bytes(void) { return (int)sizeof(ncclUniqueId); }

int tm_comm_init(tm_comm** out, int rank, int world, const void* id, int device) {
  if (!out || !id || world < 1 || rank < 0 || rank >= world) return TM_ERR_ARGUMENT;
  NcclApi& a = api();
  if (!a.ok) {
    g_comm_err = a.err;
    return TM_ERR_CUDA;
  }
  if (cudaSetDevice(device) != cudaSuccess) {
    g_comm_err = "cudaSetDevice failed";
    return TM_ERR_CUDA;
  }
  ncclUniqueId uid;
  memcpy(&uid, id, sizeof uid);
  tm_comm* c = new tm_comm();
  ncclResult_t r = a.comm_init_rank(&c->comm, world, uid, rank);
  if (r != ncclSuccess) {
    delete c;
    return comm_fail("ncclCommInitRank", r);
  }
  c->rank = rank;
  c->world = world;
  c->device = device;
  *out = c;
  return TM_OK;
}

void tm_comm_destroy(tm_comm* c) {
  if (!c) return;
  if (c->comm && api().ok) api().comm_destroy(c->comm);
  delete c;
}

// d_recv[r * bytes + i] = rank r's d_send[i]  (enqueued on `stream`)
int tm_comm_allgather(tm_comm* c, const void* d_send, void* d_recv, size_t bytes_per_rank, void* stream) {
  if (!c || (!d_send && bytes_per_rank) || (!d_recv && bytes_per_rank)) return TM_ERR_ARGUMENT;
  ncclResult_t r = api().all_gather(d_send, d_recv, bytes_per_rank, ncclUint8, c->comm, (cudaStream_t)stream);
  if (r != ncclSuccess) return comm_fail("ncclAllGather", r);
  return TM_OK;
}

}  // extern "C"
