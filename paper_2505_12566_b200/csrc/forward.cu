// forward.cu -- multi-GPU forwarding of deferred requests over peer memory
// ("transmission between models", P:561 DMA,
// P:617-619 zero-copy).
//
// After stage k every rank g holds its deferred requests as a stable compacted
// list of D_g ids (+ payload rows).  The next stage's batch is the GLOBAL
// stable list (rank-major), split into contiguous blocks over the destination
// ranks R:  block d covers global positions [lo_d, lo_{d+1}), lo_d =
// floor(d * D / |R|), D = sum_g D_g  (the same plan as dist.exchange_plan).
// Instead of a count all-gather + NCCL all-to-all with host split sizes, the
// kernels exchange counts and data through memory every rank can address
// (CUDA IPC mappings of the peers' buffers over NVLink/NVSwitch):
//   F1 fwd_publish_kernel: store {epoch, D_g} into slot g of every rank's
//      count array (system-scope release stores).
//   F2 fwd_scatter_kernel: wait (acquire) until all W counts of this epoch
//      are visible, then write every local deferred item straight into the
//      receive buffer of its destination rank at its final position
//      (j - lo_d, j = off_g + i); the last CTA to finish publishes {epoch} into
//      slot g of every rank's done array and writes this rank's receive count.
//   F3 fwd_wait_kernel: wait until all W ranks' done flags carry the epoch (the
//      receive buffer is complete; later kernels on the stream may read it).
// No host round trip, no NCCL, no split sizes on the host: the whole forward
// is stream-ordered and graph-capturable.  Epochs are caller-supplied and must
// increase per forward (flags are never reset).
#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace {

__device__ __forceinline__ void st_release_sys(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long globaltimer_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// Spin until (flag word `p`, shifted) == epoch; gives up after kFwdTimeoutNs
// (a peer that never publishes would otherwise hang the GPU), ORs
// HS_STATUS_TIMEOUT into *status and returns false.
constexpr unsigned long long kFwdTimeoutNs = 10ull * 1000 * 1000 * 1000;
__device__ __forceinline__ bool wait_epoch(const unsigned long long* p, int shift, unsigned epoch,
                                           unsigned long long* out, uint32_t* status) {
  unsigned long long v = ld_acquire_sys(p);
  const unsigned long long t0 = globaltimer_ns();
  while ((unsigned)(v >> shift) != epoch) {
    if (globaltimer_ns() - t0 > kFwdTimeoutNs) {
      if (status) atomicOr(status, HS_STATUS_TIMEOUT);
      return false;
    }
    __nanosleep(64);
    v = ld_acquire_sys(p);
  }
  *out = v;
  return true;
}

__global__ void fwd_publish_kernel(const int64_t* d_count, int64_t cap, int rank, const __grid_constant__ FwdPeers peers,
                                   unsigned epoch) {
  pdl_start();
  const int h = threadIdx.x;
  if (h >= peers.world) return;
  int64_t c = *d_count;
  c = c < 0 ? 0 : (c > cap ? cap : c);
  st_release_sys(peers.counts[h] + rank, ((unsigned long long)epoch << 32) | (unsigned long long)c);
}

// block bounds of the destination split: lo_d = floor(d * D / R)
__device__ __forceinline__ int64_t blk_lo(int64_t d, int64_t D, int64_t R) { return d * D / R; }

__global__ void __launch_bounds__(256) fwd_scatter_kernel(const int64_t* __restrict__ ids,
                                                          const uint4* __restrict__ payload,
                                                          int64_t row_vec, int rank,
                                                          const __grid_constant__ FwdPeers peers,
                                                          unsigned epoch, const __grid_constant__ FwdDest dest,
                                                          int64_t* d_recv_count, unsigned* done_ctr,
                                                          uint32_t* status) {
  pdl_start();
  __shared__ long long cnt[kFwdMaxWorld];
  __shared__ long long s_off, s_D;
  __shared__ int s_ok;
  const int W = peers.world;
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < W) {
    unsigned long long v = 0;
    if (!wait_epoch(peers.my_counts + threadIdx.x, 32, epoch, &v, status)) s_ok = 0;
    cnt[threadIdx.x] = (long long)(v & 0xFFFFFFFFull);
  }
  __syncthreads();
  if (!s_ok) return;      // timed out: nothing is written, the flag is raised
  if (threadIdx.x == 0) {
    long long off = 0, D = 0;
    for (int h = 0; h < W; ++h) {
      if (h < rank) off += cnt[h];
      D += cnt[h];
    }
    s_off = off;
    s_D = D;
  }
  __syncthreads();
  const int64_t n = cnt[rank], off = s_off, D = s_D, R = dest.n;
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  // one warp per item: lane 0 writes the id, the warp copies the payload row
  for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; i < n; i += nwarps) {
    const int64_t j = off + i;
    const int64_t d = ((j + 1) * R + D - 1) / D - 1;        // largest d with lo_d <= j
    const int h = dest.ranks[d];
    const int64_t pos = j - blk_lo(d, D, R);
    if (lane == 0) peers.recv_ids[h][pos] = ids[i];
    if (row_vec) {
      const uint4* s = payload + i * row_vec;
      uint4* t = reinterpret_cast<uint4*>(peers.recv_payload[h]) + pos * row_vec;
      for (int64_t v = lane; v < row_vec; v += 32) t[v] = ldg_stream(s + v);
    }
  }
  // completion: the last CTA publishes "done" to every rank (after all CTAs'
  // peer writes are visible system-wide) and writes this rank's receive count
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned prev = atomicAdd(done_ctr, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      *done_ctr = 0u;                                         // re-armed for the next forward
      int64_t recv = 0;
      for (int64_t d = 0; d < R; ++d)
        if (dest.ranks[d] == rank) recv += blk_lo(d + 1, D, R) - blk_lo(d, D, R);
      *d_recv_count = recv;
      for (int h = 0; h < W; ++h) st_release_sys(peers.done[h] + rank, (unsigned long long)epoch);
    }
  }
}

__global__ void fwd_wait_kernel(const unsigned long long* my_done, int world, unsigned epoch,
                                uint32_t* status) {
  pdl_start();
  const int h = threadIdx.x;
  if (h >= world) return;
  unsigned long long v;
  wait_epoch(my_done + h, 0, epoch, &v, status);
}

}  // namespace

cudaError_t launch_fwd_publish(const int64_t* d_count, int64_t cap, int rank, const FwdPeers& p,
                               unsigned epoch, cudaStream_t s) {
  return launch_pdl(fwd_publish_kernel, dim3(1), dim3(32), 0, s, d_count, cap, rank, p, epoch);
}

cudaError_t launch_fwd_scatter(const int64_t* ids, const void* payload, int64_t row_bytes, int64_t cap,
                               int rank, const FwdPeers& p, unsigned epoch, const FwdDest& dest,
                               int64_t* d_recv_count, unsigned* done_ctr, uint32_t* status,
                               cudaStream_t s) {
  const int64_t want = (cap * 32 + 255) / 256;
  int grid = (int)(want < (int64_t)num_sms() * 8 ? want : (int64_t)num_sms() * 8);
  if (grid < 1) grid = 1;
  return launch_pdl(fwd_scatter_kernel, dim3(grid), dim3(256), 0, s, ids,
                    reinterpret_cast<const uint4*>(payload), row_bytes / 16, rank, p, epoch, dest,
                    d_recv_count, done_ctr, status);
}

cudaError_t launch_fwd_wait(const unsigned long long* my_done, int world, unsigned epoch, uint32_t* status,
                            cudaStream_t s) {
  return launch_pdl(fwd_wait_kernel, dim3(1), dim3(32), 0, s, my_done, world, epoch, status);
}

}  // namespace hs
