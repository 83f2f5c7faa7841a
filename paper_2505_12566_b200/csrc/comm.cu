// comm.cu -- the library's own NCCL communicator (SURVEY 8(b) hs_comm_*) for
// request-sharded calibration across GPUs (S:212 order-independent
// merging of integer counts).
//
// NCCL is opened lazily with dlopen("libnccl.so.2") on the first
// hs_comm_* call: libhs.so has no link-time NCCL dependency, so single-GPU
// users never load it (inside a PyTorch process the already-loaded NCCL of
// the same soname is reused).  Only nccl.h's types are used at compile time.
#include <dlfcn.h>
#include <cstring>
#include <nccl.h>

#include <mutex>

#include "hs_internal.h"

struct hs_comm_s {
  ncclComm_t nc;
  int rank, world, device;
};

namespace hs {

namespace {

struct NcclApi {
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
  bool ok = false;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return;
    api.get_unique_id = reinterpret_cast<decltype(api.get_unique_id)>(dlsym(h, "ncclGetUniqueId"));
    api.comm_init_rank = reinterpret_cast<decltype(api.comm_init_rank)>(dlsym(h, "ncclCommInitRank"));
    api.comm_destroy = reinterpret_cast<decltype(api.comm_destroy)>(dlsym(h, "ncclCommDestroy"));
    api.all_reduce = reinterpret_cast<decltype(api.all_reduce)>(dlsym(h, "ncclAllReduce"));
    api.error_string = reinterpret_cast<decltype(api.error_string)>(dlsym(h, "ncclGetErrorString"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce;
  });
  return api;
}

}  // namespace

const char* nccl_error(int r) {
  const NcclApi& a = nccl();
  return a.error_string ? a.error_string((ncclResult_t)r) : "NCCL error";
}

bool nccl_available() { return nccl().ok; }

int nccl_unique_id(void* out) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  ncclUniqueId id;
  const ncclResult_t r = a.get_unique_id(&id);
  if (r == ncclSuccess) memcpy(out, &id, sizeof id);
  return (int)r;
}

int nccl_comm_create(const void* id_bytes, int rank, int world, int device, hs_comm_s** out) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  ncclUniqueId id;
  memcpy(&id, id_bytes, sizeof id);
  cudaSetDevice(device);
  hs_comm_s* c = new hs_comm_s{nullptr, rank, world, device};
  const ncclResult_t r = a.comm_init_rank(&c->nc, world, id, rank);
  if (r != ncclSuccess) {
    delete c;
    return (int)r;
  }
  *out = c;
  return 0;
}

int nccl_comm_destroy(hs_comm_s* c) {
  const NcclApi& a = nccl();
  int r = 0;
  if (a.ok && c->nc) r = (int)a.comm_destroy(c->nc);
  delete c;
  return r;
}

int nccl_allreduce_i32_sum(int32_t* buf, size_t count, hs_comm_s* c, cudaStream_t s) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  return (int)a.all_reduce(buf, buf, count, ncclInt32, ncclSum, c->nc, s);
}

}  // namespace hs
