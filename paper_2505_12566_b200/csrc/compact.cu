// compact.cu -- K3 (threshold test + stable compaction) and K4 (payload gather).
//
// The router's per-stage decision: an item is deferred to the next,
// larger model iff its confidence is below the stage threshold (ties accept;
// the last model answers everything).  The deferred items must form the next
// stage's batch in their original order, so the split is a stable partition:
// a single-pass scan with decoupled look-back (Merrill & Garland).  CTA b owns
// the 4,096-item tile b (blocks are dispatched in index order, as in CUB's
// single-pass scan), ranks its items with warp ballots, publishes its deferred
// count, and walks back over predecessor descriptors for its exclusive prefix.
// Tiles are taken from a TICKET (an atomic counter in the workspace) rather
// than from blockIdx: a CTA only ever waits on tiles whose CTAs started before
// it, so the look-back makes progress whatever order the hardware dispatches
// CTAs in and however many are resident (the CTA drawing the last ticket
// re-arms the counter for the next launch).
// Descriptors are 64-bit {epoch:32 | flag:2 | count:30}, written and read
// with relaxed gpu-scope accesses (self-contained words); the epoch (bumped by the
// last tile of every launch) makes stale descriptors from earlier launches
// read as "not ready", so there is no reset pass and no memset between calls.
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace {

constexpr unsigned long long kFlagA = 1ull << 30;   // aggregate available
constexpr unsigned long long kFlagP = 2ull << 30;   // inclusive prefix available
constexpr unsigned long long kValMask = (1ull << 30) - 1;

__device__ __forceinline__ unsigned long long* tile_status(void* ws) {
  return reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(ws) + sizeof(CompactWs));
}
// Tile of this CTA: the next ticket.  Thread 0 draws it; the CTA that draws
// the last one (every CTA of the grid has drawn) re-arms the counter.
__device__ __forceinline__ int64_t draw_tile(CompactWs* ws) {
#ifdef HS_AB_NO_TICKET
  return (int64_t)blockIdx.x;
#endif
  __shared__ unsigned s_t;
  if (threadIdx.x == 0) {
    const unsigned t = atomicAdd(&ws->ticket, 1u);
    if (t == gridDim.x - 1) ws->ticket = 0u;
    s_t = t;
  }
  __syncthreads();
  return (int64_t)s_t;
}

// Descriptor accesses: a descriptor is one self-contained 64-bit word (epoch,
// flag and count together) and no other data is read on its strength -- the
// lists are consumed by the next kernel -- so relaxed gpu-scope accesses
// suffice (a release store costs a MEMBAR on the look-back's critical path;
// HS_AB_K3_ACQREL restores acquire / release for A/B).
__device__ __forceinline__ unsigned long long desc_ld(const unsigned long long* p) {
#ifdef HS_AB_K3_ACQREL
  return ld_acquire(p);
#else
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
#endif
}
__device__ __forceinline__ void desc_st(unsigned long long* p, unsigned long long v) {
#ifdef HS_AB_K3_ACQREL
  st_release(p, v);
#else
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
#endif
}

__device__ __forceinline__ unsigned desc_flag(unsigned long long d, unsigned epoch) {
  return (unsigned)(d >> 32) == epoch ? (unsigned)((d >> 30) & 3u) : 0u;   // 0 = not ready
}

__global__ void __launch_bounds__(kCompactThreads) route_compact_kernel(const CompactArgs a) {
  pdl_start();
  constexpr int T = kCompactThreads, I = kCompactItems, NW = T / 32;
  __shared__ int s_cnt[I * NW];     // deferred count per (item row j, warp), j-major
  __shared__ int s_off[I * NW];     // exclusive offsets within the tile
  __shared__ long long s_excl;

  CompactWs* ws = reinterpret_cast<CompactWs*>(a.ws);
  unsigned long long* st = tile_status(a.ws);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;

  const int64_t tile = draw_tile(ws);
  int64_t n = a.n;
  if (a.d_n) n = min(*a.d_n, a.n);
  const int64_t ntiles = (n + kCompactTile - 1) / kCompactTile;
  if (ntiles == 0) {
    if (tile == 0 && tid == 0) {
      a.counts[0] = 0;
      a.counts[1] = 0;
    }
    return;
  }
  if (tile >= ntiles) return;
  const unsigned epoch = *(volatile unsigned*)&ws->epoch;
  const unsigned long long etag = (unsigned long long)epoch << 32;

  {
    const int64_t base = tile * kCompactTile;
    const float thr = a.sel_dest ? 0.5f : (a.d_threshold ? *a.d_threshold : a.threshold);
    // skip connections: band edges of this model's
    // successors, computed from the (possibly device-resident) threshold
    float edges[kMaxSkipEdges];
    int nedges = 0;
    if (a.skip_dest) {
      nedges = a.skip_K - 2 - a.skip_stage;   // s - 1 edges for s = K-1-k successors
      if (nedges > kMaxSkipEdges) nedges = kMaxSkipEdges;
      const int sc = nedges + 1;
      double p10 = 1.0;
#pragma unroll
      for (int e = 0; e < kMaxSkipEdges; ++e) {
        p10 *= 10.0;
        if (e < nedges)
          edges[e] = a.skip_mode == 1 ? (float)((double)thr / p10)
                                      : (float)((double)thr * (double)(sc - 1 - e) / (double)sc);
      }
    }
    // ---- all loads of the tile first (independent, coalesced: item j of thread
    //      tid is base + j*T + tid), so they overlap instead of serialising
    //      behind the ballots and the output stores
    float cv[I];
    int64_t idv[I];
    int32_t pv[I];
    const bool pred1 = a.acc_pred && a.pred_len == 1;
#pragma unroll
    for (int j = 0; j < I; ++j) {
      const int64_t i = base + (int64_t)j * T + tid;
      const bool in = i < n;
      // selection mode (skip connections): the "conf" of item i is whether
      // request i is due at model sel_k (1) or not (0)
      cv[j] = in ? (a.sel_dest ? (__ldg(a.sel_dest + i) == a.sel_k ? 0.f : 1.f) : __ldg(a.conf + i)) : 0.f;
      idv[j] = (in && a.ids) ? __ldg(a.ids + i) : i;
      pv[j] = (in && pred1) ? __ldg(a.pred + i) : 0;
    }
    bool dfr[I];
    unsigned bal[I];
#pragma unroll
    for (int j = 0; j < I; ++j) {
      const int64_t i = base + (int64_t)j * T + tid;
      // NaN confidence: deferred (unless last).  Selection mode: "deferred" =
      // selected (cv = 0 < thr = 0.5)
      const bool d = (i < n) && !(a.is_last || cv[j] >= thr);
      dfr[j] = d;
      bal[j] = __ballot_sync(0xFFFFFFFFu, d);
      if (lane == 0) s_cnt[j * NW + wid] = __popc(bal[j]);
    }
    __syncthreads();
    // ---- tile-local exclusive scan over (j, warp) in index order: warp 0
    if (wid == 0) {
      constexpr int PER = I * NW / 32;   // 4 entries per lane
      int loc[PER];
      int sum = 0;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        loc[q] = s_cnt[lane * PER + q];
        sum += loc[q];
      }
      int incl = sum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= o) incl += y;
      }
      int run = incl - sum;
#pragma unroll
      for (int q = 0; q < PER; ++q) {
        s_off[lane * PER + q] = run;
        run += loc[q];
      }
      const long long agg = __shfl_sync(0xFFFFFFFFu, incl, 31);
      // ---- decoupled look-back for the deferred count before this tile
      long long excl = 0;
      if (tile == 0) {
        if (lane == 0) desc_st(&st[0], etag | kFlagP | (unsigned long long)agg);
      } else {
        if (lane == 0) desc_st(&st[tile], etag | kFlagA | (unsigned long long)agg);
        int64_t pred = tile - 1;
        while (true) {
          const int64_t idx = pred - lane;
          unsigned long long d = (idx >= 0) ? desc_ld(&st[idx]) : (etag | kFlagP);
          while (__any_sync(0xFFFFFFFFu, desc_flag(d, epoch) == 0)) {
            if (desc_flag(d, epoch) == 0) d = desc_ld(&st[idx]);
          }
          const unsigned pm = __ballot_sync(0xFFFFFFFFu, desc_flag(d, epoch) == 2);
          long long val = (long long)(d & kValMask);
          if (pm) {
            const int first = __ffs(pm) - 1;
            excl += warp_sum(lane <= first ? val : 0ll);
            break;
          }
          excl += warp_sum(val);
          pred -= 32;
        }
        if (lane == 0) desc_st(&st[tile], etag | kFlagP | (unsigned long long)(excl + agg));
      }
      if (lane == 0 && tile == ntiles - 1) {
        // the last tile knows the totals; it also retires this launch's epoch
        a.counts[0] = n - (excl + agg);
        a.counts[1] = excl + agg;
        ws->epoch = epoch + 1u;
      }
      if (lane == 0) s_excl = excl;
    }
    __syncthreads();
    const long long excl = s_excl;
    const long long acc_base = base - excl;   // accepted items before this tile
    const unsigned lt = lanemask_lt();
#pragma unroll
    for (int j = 0; j < I; ++j) {
      const int64_t i = base + (int64_t)j * T + tid;
      if (i >= n) continue;
      const int local = j * T + tid;
      const int drank = s_off[j * NW + wid] + __popc(bal[j] & lt);
      if (a.skip_dest) {
        // next model of request idv[j]: k+1+band (deferred) or K+k (answered at k)
        int dst = a.skip_K + a.skip_stage;
        if (dfr[j]) {
          int band = 0;
#pragma unroll
          for (int e = 0; e < kMaxSkipEdges; ++e)
            if (e < nedges && !(cv[j] >= edges[e])) ++band;   // c < edge, or NaN
          dst = a.skip_stage + 1 + band;
        }
        a.skip_dest[idv[j]] = dst;
      }
      if (dfr[j]) {
        const int64_t pos = excl + drank;
        if (a.def_ids) a.def_ids[pos] = idv[j];
        if (a.def_pos) a.def_pos[pos] = i;
      } else {
        const int64_t pos = acc_base + (local - drank);
        if (a.acc_ids) a.acc_ids[pos] = idv[j];
        if (a.acc_conf) a.acc_conf[pos] = cv[j];
        if (pred1) {
          a.acc_pred[pos] = pv[j];
        } else if (a.acc_pred) {
          for (int t = 0; t < a.pred_len; ++t)
            a.acc_pred[pos * a.pred_len + t] = a.pred[i * a.pred_len + t];
        }
      }
    }
  }

}

// ---------------------------------------------------------------------------
// K3 fast path (the plain cascade split: no selection / skip modes, at most one
// prediction word per item): thread t owns the 8 consecutive items
// base + 8t .. base + 8t + 7, loaded with 128-bit loads when the tile is full
// and the arrays are 16-byte aligned.  Ranks come from a block scan of the
// per-thread deferred counts; the split is staged in shared memory in tile
// order (accepted first, then deferred) and written out coalesced.
// ---------------------------------------------------------------------------
constexpr int kFastItems = 8;
static_assert(kFastItems * kCompactThreads == kCompactTile, "one tile per CTA");

// T threads x 8 items per tile: 256 (2,048-item tiles, small batches) or 1,024
// (8,192-item tiles: 4x fewer tiles, so the look-back that decides the
// kernel's latency crosses 4x fewer descriptors; the split is staged in
// dynamic shared memory, 16 B per item).
template <int T, int I = kFastItems>
__global__ void __launch_bounds__(T) route_compact_fast_kernel(const CompactArgs a, int vec) {
  pdl_start();
  constexpr int NW = T / 32, TILE = T * I;
  static_assert(I % 4 == 0 && I <= 32, "items per thread: 128-bit loads, one mask word");
  static_assert(NW <= 32, "one warp scans the warp offsets");
  extern __shared__ __align__(16) long long s_dyn[];
  long long* s_id = s_dyn;             // accepted ids [0, A_t), deferred ids [A_t, tn)
  long long* s_aux = s_dyn + TILE;     // accepted: pred << 32 | conf bits; deferred: position
  __shared__ int s_woff[NW];
  __shared__ long long s_excl;
  __shared__ int s_agg;

  CompactWs* ws = reinterpret_cast<CompactWs*>(a.ws);
  unsigned long long* st = tile_status(a.ws);
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const bool pred1 = a.acc_pred && a.pred_len == 1;
  // The item loads are issued speculatively within the capacity a.n (the
  // buffers are capacity-sized) together with the device count and threshold,
  // so the tile's data and *d_n arrive after one memory latency, not two.
  // They are issued for tile blockIdx.x while the ticket is drawn (the CTAs
  // nearly always start, and so draw, in blockIdx order); a CTA that draws
  // another tile reloads.
  const int64_t ncap = a.n;
  float cv[I];
  int64_t idv[I];
  int32_t pv[I];
  auto load = [&](int64_t i0) {
    if (vec && i0 + I <= ncap) {
      const float4* c4 = reinterpret_cast<const float4*>(a.conf + i0);
#pragma unroll
      for (int q = 0; q < I / 4; ++q) {
        const float4 x = __ldg(c4 + q);
        cv[4 * q] = x.x; cv[4 * q + 1] = x.y; cv[4 * q + 2] = x.z; cv[4 * q + 3] = x.w;
      }
      if (a.ids) {
        const longlong2* q = reinterpret_cast<const longlong2*>(a.ids + i0);
#pragma unroll
        for (int j = 0; j < I / 2; ++j) {
          const longlong2 y = __ldg(q + j);
          idv[2 * j] = y.x;
          idv[2 * j + 1] = y.y;
        }
      } else {
#pragma unroll
        for (int j = 0; j < I; ++j) idv[j] = i0 + j;
      }
      if (pred1) {
        const int4* q = reinterpret_cast<const int4*>(a.pred + i0);
#pragma unroll
        for (int k = 0; k < I / 4; ++k) {
          const int4 x = __ldg(q + k);
          pv[4 * k] = x.x; pv[4 * k + 1] = x.y; pv[4 * k + 2] = x.z; pv[4 * k + 3] = x.w;
        }
      } else {
#pragma unroll
        for (int j = 0; j < I; ++j) pv[j] = 0;
      }
    } else {
#pragma unroll
      for (int j = 0; j < I; ++j) {
        const int64_t i = i0 + j;
        const bool in = i < ncap;
        cv[j] = in ? __ldg(a.conf + i) : 0.f;
        idv[j] = (in && a.ids) ? __ldg(a.ids + i) : i;
        pv[j] = (in && pred1) ? __ldg(a.pred + i) : 0;
      }
    }
  };
  load((int64_t)blockIdx.x * TILE + (int64_t)tid * I);
  const int64_t tile = draw_tile(ws);
  const int64_t base = tile * TILE;
  const int64_t i0 = base + (int64_t)tid * I;
  if (tile != (int64_t)blockIdx.x) load(i0);          // block-uniform, rare
  int64_t n = ncap;
  if (a.d_n) n = min(*a.d_n, ncap);
  const float thr = a.d_threshold ? *a.d_threshold : a.threshold;
  const int64_t ntiles = (n + TILE - 1) / TILE;
  if (ntiles == 0) {
    if (tile == 0 && tid == 0) {
      a.counts[0] = 0;
      a.counts[1] = 0;
    }
    return;
  }
  if (tile >= ntiles) return;
  const unsigned epoch = *(volatile unsigned*)&ws->epoch;
  const unsigned long long etag = (unsigned long long)epoch << 32;
  const int tn = (int)min((int64_t)TILE, n - base);
  // D3 per item (NaN defers; the last stage accepts all), D4 ranks
  unsigned dm = 0;
#pragma unroll
  for (int j = 0; j < I; ++j)
    dm |= (unsigned)((i0 + j < n) && !(a.is_last || cv[j] >= thr)) << j;
  const int cnt = __popc(dm);
  int incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += y;
  }
  if (lane == 31) s_woff[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int wv = lane < NW ? s_woff[lane] : 0;
    int wi = wv;
#pragma unroll
    for (int o = 1; o < NW; o <<= 1) {
      const int y = __shfl_up_sync(0xFFFFFFFFu, wi, o);
      if (lane >= o) wi += y;
    }
    if (lane < NW) s_woff[lane] = wi - wv;
    const long long agg = __shfl_sync(0xFFFFFFFFu, wi, NW - 1);
    long long excl = 0;
    if (tile == 0) {
      if (lane == 0) desc_st(&st[0], etag | kFlagP | (unsigned long long)agg);
    } else {
      if (lane == 0) desc_st(&st[tile], etag | kFlagA | (unsigned long long)agg);
      int64_t pred = tile - 1;
      while (true) {
        const int64_t idx = pred - lane;
        unsigned long long d = (idx >= 0) ? desc_ld(&st[idx]) : (etag | kFlagP);
        while (__any_sync(0xFFFFFFFFu, desc_flag(d, epoch) == 0)) {
          if (desc_flag(d, epoch) == 0) d = desc_ld(&st[idx]);
        }
        const unsigned pm = __ballot_sync(0xFFFFFFFFu, desc_flag(d, epoch) == 2);
        const long long val = (long long)(d & kValMask);
        if (pm) {
          const int first = __ffs(pm) - 1;
          excl += warp_sum(lane <= first ? val : 0ll);
          break;
        }
        excl += warp_sum(val);
        pred -= 32;
      }
      if (lane == 0) desc_st(&st[tile], etag | kFlagP | (unsigned long long)(excl + agg));
    }
    if (lane == 0) {
      if (tile == ntiles - 1) {
        a.counts[0] = n - (excl + agg);
        a.counts[1] = excl + agg;
        ws->epoch = epoch + 1u;
      }
      s_excl = excl;
      s_agg = (int)agg;
    }
  }
  __syncthreads();
  const long long excl = s_excl;
  const int nacc = tn - s_agg;
  // stage in tile order: accepted at [0, nacc), deferred at [nacc, tn)
  int dr = s_woff[wid] + incl - cnt;          // deferred items of this tile before item i0
  int ar = tid * I - dr;                      // accepted items before item i0
#pragma unroll
  for (int j = 0; j < I; ++j) {
    if (i0 + j >= n) break;
    if ((dm >> j) & 1u) {
      s_id[nacc + dr] = idv[j];
      s_aux[nacc + dr] = i0 + j;
      ++dr;
    } else {
      s_id[ar] = idv[j];
      s_aux[ar] = ((long long)(uint32_t)pv[j] << 32) | (long long)__float_as_uint(cv[j]);
      ++ar;
    }
  }
  __syncthreads();
  const int64_t acc_base = base - excl;       // accepted items before this tile
  for (int p = tid; p < tn; p += T) {
    const long long id = s_id[p], aux = s_aux[p];
    if (p < nacc) {
      const int64_t pos = acc_base + p;
      if (a.acc_ids) a.acc_ids[pos] = id;
      if (a.acc_conf) a.acc_conf[pos] = __uint_as_float((uint32_t)aux);
      if (pred1) a.acc_pred[pos] = (int32_t)(aux >> 32);
    } else {
      const int64_t pos = excl + (p - nacc);
      if (a.def_ids) a.def_ids[pos] = id;
      if (a.def_pos) a.def_pos[pos] = aux;
    }
  }
}

// K4: dst[j] = src[pos[j]] for j < *d_count, rows of row_bytes (multiple of 16)
__global__ void __launch_bounds__(256) gather_rows_kernel(const int64_t* __restrict__ pos,
                                                          const int64_t* d_count, int64_t cap,
                                                          const uint4* __restrict__ src,
                                                          int64_t row_vec, uint4* __restrict__ dst) {
  pdl_start();
  int64_t n = cap;
  if (d_count) n = min(*d_count, cap);
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t j = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; j < n; j += nwarps) {
    const uint4* s = src + pos[j] * row_vec;
    uint4* d = dst + j * row_vec;
    int64_t v = lane;
    for (; v + 96 < row_vec; v += 128) {
      const uint4 x0 = ldg_stream(s + v), x1 = ldg_stream(s + v + 32), x2 = ldg_stream(s + v + 64),
                  x3 = ldg_stream(s + v + 96);
      d[v] = x0;
      d[v + 32] = x1;
      d[v + 64] = x2;
      d[v + 96] = x3;
    }
    for (; v < row_vec; v += 32) d[v] = ldg_stream(s + v);
  }
}

// Count of the items the threshold test defers (the next stage's batch size),
// without the compaction: lets the next stage's confidence start while the
// compaction of this stage runs off the critical path.  One atomic per CTA into
// *out (zero-filled by the caller).
__global__ void __launch_bounds__(256) count_deferred_kernel(const float* __restrict__ conf, int64_t cap,
                                                             const int64_t* d_n, float threshold,
                                                             const float* d_threshold, int is_last,
                                                             unsigned long long* out) {
  pdl_start();
  __shared__ unsigned s_c[8];
  int64_t n = cap;
  if (d_n) n = min(*d_n, cap);
  const float thr = d_threshold ? *d_threshold : threshold;
  unsigned c = 0;
  if (!is_last) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x * 4;
    for (int64_t i = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) * 4; i < n; i += stride) {
      if (i + 4 <= n) {
        const float4 v = __ldg(reinterpret_cast<const float4*>(conf + i));
        c += !(v.x >= thr) + !(v.y >= thr) + !(v.z >= thr) + !(v.w >= thr);
      } else {
        for (int64_t j = i; j < n; ++j) c += !(__ldg(conf + j) >= thr);
      }
    }
  }
  c = __reduce_add_sync(0xFFFFFFFFu, c);
  if ((threadIdx.x & 31) == 0) s_c[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t += s_c[w];
    if (t) atomicAdd(out, (unsigned long long)t);
  }
}

}  // namespace

cudaError_t launch_count_deferred(const float* conf, int64_t cap, const int64_t* d_n, float threshold,
                                  const float* d_threshold, int is_last, unsigned long long* out,
                                  cudaStream_t s) {
  const int64_t want = (cap + 1023) / 1024;
  const int64_t lim = (int64_t)num_sms() * 2;
  const int grid = (int)(want < 1 ? 1 : (want < lim ? want : lim));
  return launch_pdl(count_deferred_kernel, dim3(grid), dim3(256), 0, s, conf, cap, d_n, threshold,
                    d_threshold, is_last, out);
}

size_t compact_ws_bytes(int64_t n) {
  const int64_t tiles = (n + kCompactTile - 1) / kCompactTile;
  return sizeof(CompactWs) + (size_t)(tiles > 0 ? tiles : 1) * sizeof(unsigned long long);
}

static bool aligned16(const void* p) { return ((uintptr_t)p & 15u) == 0; }

cudaError_t launch_route_compact(const CompactArgs& a, cudaStream_t s) {
  const int64_t tiles = (a.n + kCompactTile - 1) / kCompactTile;
  const int grid = (int)(tiles > 0 ? tiles : 1);
  const bool fast = !a.sel_dest && !a.skip_dest && (!a.acc_pred || a.pred_len == 1);
  if (fast) {
    const int vec = aligned16(a.conf) && aligned16(a.ids) && (!a.acc_pred || aligned16(a.pred));
    // tile size (A/B on one box, five-stage C2 step in a graph): 4,096 items
    // (512 threads, 64 KB staging) 323.8 us; 8,192 items (1,024 threads, 128 KB)
    // 338.4 us; 2,048 items (256 threads) 360.3 us.  The 128 KB CTAs hold SM
    // slots the next stage's K1 needs while it launches early; the 2,048-item
    // grid is 4x larger.  HS_COMPACT_TILES=8192 / 2048 select the others.
    static const int tiles_env = [] {
      const char* e = getenv("HS_COMPACT_TILES");
      if (getenv("HS_COMPACT_SMALL_TILES") && getenv("HS_COMPACT_SMALL_TILES")[0] == '1') return 2048;
      return e ? atoi(e) : 4096;
    }();
    static const bool mid_ok = cudaFuncSetAttribute(route_compact_fast_kernel<512>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    512 * kFastItems * 16) == cudaSuccess;
    static const bool big_ok = cudaFuncSetAttribute(route_compact_fast_kernel<1024>,
                                                    cudaFuncAttributeMaxDynamicSharedMemorySize,
                                                    1024 * kFastItems * 16) == cudaSuccess;
    if (tiles_env == 8192 && big_ok && a.n >= 4 * 1024 * kFastItems) {   // >= 4 tiles
      const int64_t bt = (a.n + 1024 * kFastItems - 1) / (1024 * kFastItems);
      return launch_pdl(route_compact_fast_kernel<1024>, dim3((unsigned)bt), dim3(1024),
                        (size_t)1024 * kFastItems * 16, s, a, vec);
    }
    static const bool t256 = [] {    // A/B: 4,096-item tiles from 256 threads x 16 items
      const char* e = getenv("HS_COMPACT_T256");
      return e && e[0] == '1' &&
             cudaFuncSetAttribute(route_compact_fast_kernel<256, 16>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                  256 * 16 * 16) == cudaSuccess;
    }();
    if (t256 && a.n >= 4 * 4096) {
      const int64_t mt = (a.n + 4095) / 4096;
      return launch_pdl(route_compact_fast_kernel<256, 16>, dim3((unsigned)mt), dim3(256), (size_t)256 * 16 * 16,
                        s, a, vec);
    }
    if (tiles_env == 4096 && mid_ok && a.n >= 4 * 512 * kFastItems) {
      const int64_t mt = (a.n + 512 * kFastItems - 1) / (512 * kFastItems);
      return launch_pdl(route_compact_fast_kernel<512>, dim3((unsigned)mt), dim3(512),
                        (size_t)512 * kFastItems * 16, s, a, vec);
    }
    return launch_pdl(route_compact_fast_kernel<256>, dim3(grid), dim3(256), (size_t)256 * kFastItems * 16, s,
                      a, vec);
  }
  return launch_pdl(route_compact_kernel, dim3(grid), dim3(kCompactThreads), 0, s, a);
}

cudaError_t launch_gather_rows(const int64_t* pos, const int64_t* d_count, int64_t cap,
                               const void* src, int64_t row_bytes, void* dst, cudaStream_t s) {
  if (cap <= 0 || row_bytes <= 0) return cudaSuccess;
  const int64_t want = (cap + 7) / 8;
  const int64_t lim = (int64_t)num_sms() * 8;
  const int grid = (int)(want < lim ? want : lim);
  return launch_pdl(gather_rows_kernel, dim3(grid), dim3(256), 0, s, pos, d_count, cap,
                    reinterpret_cast<const uint4*>(src), row_bytes / 16, reinterpret_cast<uint4*>(dst));
}

}  // namespace hs
