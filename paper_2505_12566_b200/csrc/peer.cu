// peer.cu -- the multi-GPU exchange of the cascade over peer memory: forwarding
// of deferred requests ("transmission between models",
// P:561 DMA, P:617-619 zero-copy) and the calibration histogram exchange
// (calib.cu's resident kernel pushes into the regions defined here).
//
// Every rank owns one PEER REGION (one exportable allocation, hs_ipc_alloc),
// mapped into every other rank's process with CUDA IPC; hs_peer_t carries the
// W region pointers as seen by this process.  Region layout (identical on
// every rank; PeerLayout):
//   header  fwd_counts[8]  {epoch:32 | count:32} written by rank g into slot g
//           fwd_done[8]    epoch written by rank g into slot g
//           cal_arrive[2]  pushes received per round parity (monotonic)
//           local words    fwd_epoch, completion counter, timeout flag,
//                          calibration round counter (this rank only)
//   cal     u64 [2][W][2^q + 2]   packed bins pushed by every rank, per parity
//   recv    int64 [2][W * cap]    receive sets of forwarded ids
//   pay     u8 [2][W * cap * P]   receive sets of payload rows
//
// Forwarding after stage k (every rank g holds D_g deferred ids in stable
// order; the next batch is the global rank-major list split into contiguous
// blocks over the destination ranks R: block d = global positions
// [floor(d*D/|R|), floor((d+1)*D/|R|)), D = sum_g D_g -- dist.exchange_plan):
//   F1 peer_publish_kernel: e = ++fwd_epoch; store {e, D_g} into slot g of
//      every rank's fwd_counts (system-scope release).
//   F2 peer_scatter_kernel: wait (acquire) for all W counts of epoch e; then
//      ONE THREAD PER ITEM writes its id at its final position in the
//      destination's receive set (consecutive items -> consecutive addresses:
//      coalesced NVLink stores), payload rows as a flat 16-byte vector copy;
//      the last CTA to finish (completion counter) writes this rank's receive
//      count and stores e into slot g of every rank's fwd_done.
//   F3 peer_wait_kernel: wait until all W done flags carry e (the receive set
//      is complete for the next stage's kernels).
// The epoch lives on the device, so the forward is graph-replayable; the
// receive set is chosen by the caller (stage parity), so the next stage's
// pointers are static.  Every wait gives up after 10 s (HS_STATUS_TIMEOUT)
// instead of hanging the GPU.
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
constexpr unsigned long long kPeerTimeoutNs = 10ull * 1000 * 1000 * 1000;

// Spin until (word >> shift) == epoch (32-bit compare); false after the timeout.
__device__ __forceinline__ bool wait_epoch(const unsigned long long* p, int shift, unsigned epoch,
                                           unsigned long long* out, uint32_t* status) {
  unsigned long long v = ld_acquire_sys(p);
  const unsigned long long t0 = globaltimer_ns();
  while ((unsigned)(v >> shift) != epoch) {
    if (globaltimer_ns() - t0 > kPeerTimeoutNs) {
      if (status) atomicOr(status, HS_STATUS_TIMEOUT);
      return false;
    }
    __nanosleep(64);
    v = ld_acquire_sys(p);
  }
  *out = v;
  return true;
}

__global__ void peer_publish_kernel(const int64_t* d_count, int64_t cap, const __grid_constant__ PeerArgs g,
                                    uint32_t* status) {
  pdl_start();
  __shared__ unsigned s_e;
  PeerHeader* me = g.hdr[g.rank];
  if (threadIdx.x == 0) s_e = me->fwd_epoch + 1u;
  __syncthreads();
  const unsigned e = s_e;
  const int h = threadIdx.x;
  if (h < g.world) {
    int64_t c = *d_count;
    if (c > cap && h == 0 && status) atomicOr(status, HS_STATUS_OVERFLOW);   // more than the regions hold
    c = c < 0 ? 0 : (c > cap ? cap : c);
    st_release_sys(&g.hdr[h]->fwd_counts[g.rank], ((unsigned long long)e << 32) | (unsigned long long)c);
  }
  __syncthreads();
  if (threadIdx.x == 0) me->fwd_epoch = e;
}

// block bounds of the destination split: lo_d = floor(d * D / R)
__device__ __forceinline__ int64_t blk_lo(int64_t d, int64_t D, int64_t R) { return d * D / R; }

__global__ void __launch_bounds__(256) peer_scatter_kernel(const int64_t* __restrict__ ids,
                                                           const uint4* __restrict__ payload,
                                                           int64_t row_vec, int set,
                                                           const __grid_constant__ PeerArgs g,
                                                           const __grid_constant__ PeerDest dest,
                                                           int64_t* d_recv_count, uint32_t* status) {
  pdl_start();
  __shared__ long long cnt[kPeerMaxWorld];
  __shared__ long long s_off, s_D;
  __shared__ int s_ok;
  const int W = g.world, rank = g.rank;
  PeerHeader* me = g.hdr[rank];
  const unsigned e = me->fwd_epoch;          // incremented by this rank's publish
  if (threadIdx.x == 0) s_ok = 1;
  __syncthreads();
  if (threadIdx.x < W) {
    unsigned long long v = 0;
    if (!wait_epoch(&me->fwd_counts[threadIdx.x], 32, e, &v, status)) s_ok = 0;
    cnt[threadIdx.x] = (long long)(v & 0xFFFFFFFFull);
  }
  __syncthreads();
  const bool ok = s_ok != 0;
  if (ok && threadIdx.x == 0) {
    long long off = 0, D = 0;
    for (int h = 0; h < W; ++h) {
      if (h < rank) off += cnt[h];
      D += cnt[h];
    }
    s_off = off;
    s_D = D;
  }
  __syncthreads();
  if (ok) {
    const int64_t n = cnt[rank], off = s_off, D = s_D, R = dest.n;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int64_t t0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    // ids: one thread per item, consecutive items land at consecutive positions
    for (int64_t i = t0; i < n; i += stride) {
      const int64_t j = off + i;
      const int64_t d = ((j + 1) * R + D - 1) / D - 1;        // largest d with lo_d <= j
      const int64_t pos = j - blk_lo(d, D, R);
      g.recv_ids[dest.ranks[d]][(int64_t)set * g.recv_stride + pos] = ids[i];
    }
    // payload: a flat copy of n * row_vec 16-byte vectors
    if (row_vec) {
      const int64_t nv = n * row_vec;
      for (int64_t v = t0; v < nv; v += stride) {
        const int64_t i = v / row_vec, c = v - i * row_vec;
        const int64_t j = off + i;
        const int64_t d = ((j + 1) * R + D - 1) / D - 1;
        const int64_t pos = j - blk_lo(d, D, R);
        uint4* t = reinterpret_cast<uint4*>(g.recv_payload[dest.ranks[d]]) +
                   ((int64_t)set * g.recv_stride + pos) * row_vec + c;
        *t = ldg_stream(payload + v);
      }
    }
  }
  // completion: every CTA arrives (also after a timeout, so the counter always
  // returns to 0); the last one publishes "done" unless some CTA timed out
  __threadfence_system();
  __syncthreads();
  if (threadIdx.x == 0) {
    if (!ok) {
      atomicExch(&me->fwd_failed, 1u);
      __threadfence();                                        // visible before the arrival below
    }
    const unsigned prev = atomicAdd(&me->fwd_ctr, 1u);
    if (prev == gridDim.x - 1) {
      __threadfence_system();
      me->fwd_ctr = 0u;                                       // re-armed for the next forward
      const unsigned failed = atomicExch(&me->fwd_failed, 0u);
      if (!failed) {
        const int64_t D = s_D, R = dest.n;
        int64_t recv = 0;
        for (int64_t d = 0; d < R; ++d)
          if (dest.ranks[d] == rank) recv += blk_lo(d + 1, D, R) - blk_lo(d, D, R);
        *d_recv_count = recv;
        for (int h = 0; h < W; ++h) st_release_sys(&g.hdr[h]->fwd_done[rank], (unsigned long long)e);
      } else {
        *d_recv_count = 0;
      }
    }
  }
}

__global__ void peer_wait_kernel(const __grid_constant__ PeerArgs g, uint32_t* status) {
  pdl_start();
  const PeerHeader* me = g.hdr[g.rank];
  const unsigned e = me->fwd_epoch;
  const int h = threadIdx.x;
  if (h >= g.world) return;
  unsigned long long v;
  wait_epoch(&me->fwd_done[h], 0, e, &v, status);
}

}  // namespace

PeerLayout peer_layout(int world, int64_t cap, int64_t payload_row_bytes, int q) {
  auto up = [](size_t x) { return (x + 255) / 256 * 256; };
  PeerLayout L{};
  const size_t nb = (q >= 1 && q <= 14) ? ((size_t)1 << q) + 2 : 0;
  L.cal_off = up(sizeof(PeerHeader));
  L.cal_words = nb;
  L.recv_off = up(L.cal_off + 2 * (size_t)world * nb * sizeof(unsigned long long));
  L.recv_stride = (size_t)world * (size_t)(cap < 0 ? 0 : cap);
  L.pay_off = up(L.recv_off + 2 * L.recv_stride * sizeof(int64_t));
  L.bytes = up(L.pay_off + 2 * L.recv_stride * (size_t)(payload_row_bytes < 0 ? 0 : payload_row_bytes));
  return L;
}

cudaError_t launch_peer_publish(const int64_t* d_count, int64_t cap, const PeerArgs& g, uint32_t* status,
                                cudaStream_t s) {
  return launch_pdl(peer_publish_kernel, dim3(1), dim3(32), 0, s, d_count, cap, g, status);
}

cudaError_t launch_peer_scatter(const int64_t* ids, const void* payload, int64_t row_bytes, int64_t cap,
                                int set, const PeerArgs& g, const PeerDest& dest, int64_t* d_recv_count,
                                uint32_t* status, cudaStream_t s) {
  // enough threads for one id (or one payload vector) each, up to 4 CTAs per SM
  const int64_t work = cap * (row_bytes ? row_bytes / 16 : 1);
  int64_t want = (work + 255) / 256;
  const int64_t cap_grid = (int64_t)num_sms() * 4;
  int grid = (int)(want < cap_grid ? want : cap_grid);
  if (grid < 1) grid = 1;
  return launch_pdl(peer_scatter_kernel, dim3(grid), dim3(256), 0, s, ids,
                    reinterpret_cast<const uint4*>(payload), row_bytes / 16, set, g, dest, d_recv_count,
                    status);
}

cudaError_t launch_peer_wait(const PeerArgs& g, uint32_t* status, cudaStream_t s) {
  return launch_pdl(peer_wait_kernel, dim3(1), dim3(32), 0, s, g, status);
}

}  // namespace hs
