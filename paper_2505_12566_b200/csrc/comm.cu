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
  ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*group_start)() = nullptr;
  ncclResult_t (*group_end)() = nullptr;
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
    api.all_gather = reinterpret_cast<decltype(api.all_gather)>(dlsym(h, "ncclAllGather"));
    api.send = reinterpret_cast<decltype(api.send)>(dlsym(h, "ncclSend"));
    api.recv = reinterpret_cast<decltype(api.recv)>(dlsym(h, "ncclRecv"));
    api.group_start = reinterpret_cast<decltype(api.group_start)>(dlsym(h, "ncclGroupStart"));
    api.group_end = reinterpret_cast<decltype(api.group_end)>(dlsym(h, "ncclGroupEnd"));
    api.ok = api.get_unique_id && api.comm_init_rank && api.comm_destroy && api.all_reduce &&
             api.all_gather && api.send && api.recv && api.group_start && api.group_end;
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
  int prev = 0;
  cudaGetDevice(&prev);                      // NCCL binds the communicator to the current device
  cudaSetDevice(device);
  hs_comm_s* c = new hs_comm_s{nullptr, rank, world, device};
  const ncclResult_t r = a.comm_init_rank(&c->nc, world, id, rank);
  cudaSetDevice(prev);                       // the caller's current device is unchanged
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

int nccl_world(const hs_comm_s* c) { return c->world; }
int nccl_rank(const hs_comm_s* c) { return c->rank; }

int nccl_allgather_i64(const int64_t* mine, int64_t* all, int64_t count, hs_comm_s* c, cudaStream_t s) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  return (int)a.all_gather(mine, all, (size_t)count, ncclInt64, c->nc, s);
}

// grouped point-to-point exchange: send[h] elements from sbuf + soff[h] to rank h,
// recv[h] elements into rbuf + roff[h] from rank h (bytes, ncclUint8)
int nccl_exchange(const char* sbuf, const int64_t* soff, const int64_t* scnt, char* rbuf,
                  const int64_t* roff, const int64_t* rcnt, int64_t elem_bytes, hs_comm_s* c,
                  cudaStream_t s) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  ncclResult_t r = a.group_start();
  for (int h = 0; h < c->world && r == ncclSuccess; ++h) {
    if (scnt[h]) r = a.send(sbuf + soff[h] * elem_bytes, (size_t)(scnt[h] * elem_bytes), ncclUint8, h, c->nc, s);
    if (r == ncclSuccess && rcnt[h])
      r = a.recv(rbuf + roff[h] * elem_bytes, (size_t)(rcnt[h] * elem_bytes), ncclUint8, h, c->nc, s);
  }
  const ncclResult_t e = a.group_end();
  return (int)(r != ncclSuccess ? r : e);
}

int nccl_allreduce_i32_sum(int32_t* buf, size_t count, hs_comm_s* c, cudaStream_t s) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  return (int)a.all_reduce(buf, buf, count, ncclInt32, ncclSum, c->nc, s);
}

int nccl_allreduce_i64_sum(int64_t* buf, size_t count, hs_comm_s* c, cudaStream_t s) {
  const NcclApi& a = nccl();
  if (!a.ok) return -1;
  return (int)a.all_reduce(buf, buf, count, ncclInt64, ncclSum, c->nc, s);
}

}  // namespace hs
