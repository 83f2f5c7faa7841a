// calib.cu -- K5 (calibration histogram) and K6 (threshold select).
//
// Offline Accuracy-Preserving threshold calibration (Alg. 1 and
// the AP mode; exact deterministic sweep of DESIGN.md reading G8): thresholds
// live on a 2^q grid, bin(c) = min(B, floor(c * B)) (exact in fp32, so
// bin(c) >= b  <=>  c >= b/B), NaN confidences never accepted.
// Round k (one model) over the validation samples still alive:
//   K5: one pass builds a shared-memory-privatised histogram over bin(c_k) of
//       (count, correct_k, correct_K) in three u32 arrays (native 32-bit
//       shared atomics), warp-aggregated with __match_any_sync for the skewed
//       bins near c = 1; CTAs merge through DSMEM (one cluster) or global
//       int32 atomics (many CTAs).
//   K6: one CTA: suffix scan over the B+2 bins and
//       b_k = min{ b : A + G + S(b) >= tau } (S is not monotone: every b is
//       examined), then A += committed correct answers; reach/handled counts.
// Histograms are integers, so a request-sharded calibration sums them across
// GPUs (all-reduce) and every rank selects the same b_k.
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace cg = cooperative_groups;

#ifdef HS_CALIB_TRACE
__device__ unsigned long long g_calib_trace[64];
#endif

namespace {

__device__ __forceinline__ int bin_of(float c, int q) {
  if (c != c) return -1;
  const float B = (float)(1 << q);
  float f = floorf(c * B);          // exact: c * 2^q
  f = fminf(fmaxf(f, 0.f), B);
  return (int)f;
}

__global__ void calib_init_kernel(CalibState* st, int32_t* hist, int nwords, long long target) {
  pdl_start();
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) {
    st->A = 0;
    st->tau = target < 0 ? 0 : target;
    st->tau_ap = target < 0 ? 1 : 0;
  }
}

// hist layout: int32 [3][B+2]; index 0 = NaN bin (never accepted), index b+1 = bin b.
// Build this CTA's share of round `round` in shared memory: samples r = start,
// start + stride, ...  Three u32 arrays (count, correct_k, correct_K per bin):
// native 32-bit shared atomics (a 64-bit shared add would be a CAS loop).
__device__ __forceinline__ void hist_zero(unsigned* sh, int q) {
  const int words = 3 * ((1 << q) + 2);
  uint4* sh4 = reinterpret_cast<uint4*>(sh);
  for (int i = threadIdx.x; i < words / 4; i += blockDim.x) sh4[i] = make_uint4(0, 0, 0, 0);
  for (int i = (words / 4) * 4 + threadIdx.x; i < words; i += blockDim.x) sh[i] = 0u;
}

// Accumulate samples r = start, start + stride, ... of round `round` into the
// shared-memory histogram `sh` -- this CTA's, or (cluster kernel) rank 0's
// through distributed shared memory.  No zeroing, no trailing barrier.
__device__ __forceinline__ void hist_accumulate(const float* __restrict__ conf,
                                                const uint8_t* __restrict__ correct, int K,
                                                int64_t N, int q, int round, const int32_t* b_idx,
                                                unsigned* sh, int64_t start, int64_t stride) {
  __shared__ int s_b[16];
  const int nb = (1 << q) + 2;
  if (threadIdx.x < 16) s_b[threadIdx.x] = threadIdx.x < round ? b_idx[threadIdx.x] : 0;
  __syncthreads();

  const uint8_t* ck = correct + (int64_t)round * N;
  const uint8_t* cK = correct + (int64_t)(K - 1) * N;
  const float* ckconf = conf + (int64_t)round * N;
  // loop bound is warp-uniform so __match_any_sync sees full warps
  const int64_t Nup = (N + 31) & ~(int64_t)31;
  for (int64_t r = start; r < Nup; r += stride) {
    const bool in = r < N;
    const int64_t rr = in ? r : 0;
    // this round's loads first; earlier rounds' confidences decide "alive"
    const float cnow = __ldg(ckconf + rr);
    const bool okk = __ldg(ck + rr) != 0;
    const bool okK0 = __ldg(cK + rr) != 0;
    bool alive = in;
    const float* cp = conf + rr;
#pragma unroll 4
    for (int j = 0; j < round; ++j, cp += N) alive &= bin_of(__ldg(cp), q) < s_b[j];
    const int key = alive ? bin_of(cnow, q) + 1 : -1;   // -1: not counted
    const bool okK = alive && okK0;
    // warp aggregation: lanes with the same bin add once, through their leader
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
    const unsigned bk = __ballot_sync(0xFFFFFFFFu, alive && okk);
    const unsigned bK = __ballot_sync(0xFFFFFFFFu, okK);
    if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) {
      atomicAdd(&sh[key], (unsigned)__popc(peers));
      const unsigned nk = __popc(peers & bk), nK = __popc(peers & bK);
      if (nk) atomicAdd(&sh[nb + key], nk);
      if (nK) atomicAdd(&sh[2 * nb + key], nK);
    }
  }
}

__device__ __forceinline__ void hist_local(const float* __restrict__ conf,
                                           const uint8_t* __restrict__ correct, int K, int64_t N,
                                           int q, int round, const int32_t* b_idx,
                                           unsigned* sh, int64_t start, int64_t stride) {
  hist_zero(sh, q);
  hist_accumulate(conf, correct, K, N, q, round, b_idx, sh, start, stride);
  __syncthreads();
}

// Add a shared-memory histogram into the global int32 [3][B+2] one.
__device__ __forceinline__ void hist_flush(const unsigned* sh, int q, int32_t* hist) {
  const int nb = (1 << q) + 2;
  for (int i = threadIdx.x; i < 3 * nb; i += blockDim.x) {
    const unsigned v = sh[i];
    if (v) atomicAdd(&hist[i], (int32_t)v);
  }
}

// One CTA's share (grid-stride) of round `round`, added into the global histogram.
__device__ __forceinline__ void hist_body(const float* __restrict__ conf,
                                          const uint8_t* __restrict__ correct, int K, int64_t N,
                                          int q, int round, const int32_t* b_idx,
                                          int32_t* __restrict__ hist, unsigned* sh) {
  hist_local(conf, correct, K, N, q, round, b_idx, sh,
             (int64_t)blockIdx.x * blockDim.x + threadIdx.x, (int64_t)gridDim.x * blockDim.x);
  hist_flush(sh, q, hist);
}

__global__ void __launch_bounds__(512) calib_hist_kernel(const float* __restrict__ conf,
                                                         const uint8_t* __restrict__ correct,
                                                         int K, int64_t N, int q, int round,
                                                         const int32_t* __restrict__ b_idx,
                                                         int32_t* __restrict__ hist) {
  pdl_start();
  extern __shared__ unsigned sh[];
  hist_body(conf, correct, K, N, q, round, b_idx, hist, sh);
}

// Histogram readers for the select: the int32 [3][B+2] global layout, or the
// u32 shared-memory layout of the cluster kernel.
struct Bin3 { long long cnt, ck, cK; };
struct GlobalHist {
  const int32_t* h;
  int nb;
  __device__ __forceinline__ Bin3 operator()(int i) const {
    return Bin3{h[i], h[nb + i], h[2 * nb + i]};
  }
};
struct SharedHist {
  const unsigned* h;
  int nb;
  __device__ __forceinline__ Bin3 operator()(int i) const {
    return Bin3{(long long)h[i], (long long)h[nb + i], (long long)h[2 * nb + i]};
  }
};

// One CTA of NT threads picks b_k (D5): thread t owns the contiguous bins
// [lo, hi) of 0..B (histogram index b+1; index 0 = NaN, never accepted).
//   pass 1: segment sums -> block totals (reach_k, G) and the suffix S(hi)
//   pass 2: smallest feasible b of each segment -> block min = b_k
//   pass 3: committed (bin >= b_k) and surviving (bin < b_k) sums
// Cross-warp steps go through warp 0 (one shuffle scan), so no thread loops
// over all warps.  Counts fit int32 (N < 2^31); feasibility is tested in int64.
template <int NT, typename Hist>
__device__ __forceinline__ void select_core(const Hist& H, int K, int q, int round,
                                            int32_t* b_idx, float* thr, int64_t* reach,
                                            int64_t* handled, int64_t* correct_total,
                                            CalibState* st) {
  constexpr int NW = NT / 32;
  static_assert(NW <= 32, "one warp scans the warp totals");
  __shared__ int sh_x[NW], sh_y[NW], sh_z[NW], sh_u[NW];
  __shared__ int sh_tot[2];
  __shared__ int sh_bk;
  __shared__ long long sh_tau, sh_A;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B = 1 << q;
  const int per = (B + 1 + NT - 1) / NT;
  const int lo = min(tid * per, B + 1), hi = min(lo + per, B + 1);

  // ---- pass 1
  int segH = 0, segCnt = 0, segK = 0;
  for (int b = lo; b < hi; ++b) {
    const Bin3 x = H(b + 1);
    segH += (int)(x.ck - x.cK);
    segCnt += (int)x.cnt;
    segK += (int)x.cK;
  }
  if (tid == 0) {                     // NaN bin: alive, never accepted
    const Bin3 x = H(0);
    segCnt += (int)x.cnt;
    segK += (int)x.cK;
  }
  int incl = segH;                    // inclusive suffix within the warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_down_sync(0xFFFFFFFFu, incl, o);
    if (lane + o < 32) incl += y;
  }
  const int wc = __reduce_add_sync(0xFFFFFFFFu, segCnt);
  const int wk = __reduce_add_sync(0xFFFFFFFFu, segK);
  if (lane == 0) {
    sh_x[wid] = incl;                 // warp total of H
    sh_y[wid] = wc;
    sh_z[wid] = wk;
  }
  __syncthreads();
  if (wid == 0) {
    const int h = lane < NW ? sh_x[lane] : 0;
    int suf = h;                      // inclusive suffix over warps
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_down_sync(0xFFFFFFFFu, suf, o);
      if (lane + o < 32) suf += y;
    }
    const int tc = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_y[lane] : 0);
    const int tk = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_z[lane] : 0);
    if (lane < NW) sh_u[lane] = suf - h;   // H of all warps after this one
    if (lane == 0) {
      sh_tot[0] = tc;
      sh_tot[1] = tk;
      if (round == 0 && st->tau_ap) st->tau = tk;   // AP: tau = correct answers of m_K
      sh_tau = st->tau;
      sh_A = st->A;
    }
  }
  __syncthreads();
  const long long reach_k = sh_tot[0], G = sh_tot[1], tau = sh_tau, A = sh_A;
  // ---- pass 2: S(b) for b in [lo, hi) built downward from S(hi)
  int best = B + 1;
  {
    long long S = (long long)sh_u[wid] + (incl - segH);
    for (int b = hi - 1; b >= lo; --b) {
      const Bin3 x = H(b + 1);
      S += x.ck - x.cK;
      if (A + G + S >= tau) best = b;
    }
  }
  best = (int)__reduce_min_sync(0xFFFFFFFFu, (unsigned)best);
  if (lane == 0) sh_x[wid] = best;
  __syncthreads();
  if (wid == 0) {
    const unsigned v = lane < NW ? (unsigned)sh_x[lane] : (unsigned)(B + 1);
    const int bk = (int)__reduce_min_sync(0xFFFFFFFFu, v);
    if (lane == 0) sh_bk = bk;   // b = B+1 (defer all) is feasible by induction
  }
  __syncthreads();
  const int bk = sh_bk;
  // ---- pass 3
  int s_ck = 0, s_cnt = 0, s_bc = 0, s_bK = 0;
  for (int b = lo; b < hi; ++b) {
    const Bin3 x = H(b + 1);
    if (b >= bk) {
      s_ck += (int)x.ck;
      s_cnt += (int)x.cnt;
    } else {
      s_bc += (int)x.cnt;
      s_bK += (int)x.cK;
    }
  }
  if (tid == 0) {
    const Bin3 x = H(0);
    s_bc += (int)x.cnt;
    s_bK += (int)x.cK;
  }
  s_ck = __reduce_add_sync(0xFFFFFFFFu, s_ck);
  s_cnt = __reduce_add_sync(0xFFFFFFFFu, s_cnt);
  s_bc = __reduce_add_sync(0xFFFFFFFFu, s_bc);
  s_bK = __reduce_add_sync(0xFFFFFFFFu, s_bK);
  if (lane == 0) {
    sh_x[wid] = s_ck;
    sh_y[wid] = s_cnt;
    sh_z[wid] = s_bc;
    sh_u[wid] = s_bK;
  }
  __syncthreads();
  if (wid == 0) {
    const int ck = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_x[lane] : 0);
    const int cnt = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_y[lane] : 0);
    const int bc = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_z[lane] : 0);
    const int bK = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_u[lane] : 0);
    if (lane == 0) {
      long long Anew = A + ck;
      b_idx[round] = bk;
      thr[round] = bk <= B ? (float)bk / (float)B : INFINITY;
      reach[round] = reach_k;
      handled[round] = cnt;
      if (round == K - 2) {
        reach[K - 1] = bc;
        handled[K - 1] = bc;
        Anew += bK;
        thr[K - 1] = 0.f;
        *correct_total = Anew;
      }
      st->A = Anew;
    }
  }
  __syncthreads();
}

template <int NT>
__device__ __forceinline__ void select_body(int K, int q, int round, int32_t* b_idx, float* thr,
                                            int64_t* reach, int64_t* handled,
                                            int64_t* correct_total, CalibState* st,
                                            int32_t* hist) {
  const int nb = (1 << q) + 2;
  select_core<NT>(GlobalHist{hist, nb}, K, q, round, b_idx, thr, reach, handled, correct_total, st);
  for (int i = threadIdx.x; i < 3 * nb; i += NT) hist[i] = 0;
  __syncthreads();
}

__global__ void __launch_bounds__(256) calib_select_kernel(int K, int q, int round,
                                                            int32_t* b_idx, float* thr,
                                                            int64_t* reach, int64_t* handled,
                                                            int64_t* correct_total,
                                                            CalibState* st, int32_t* hist) {
  pdl_start();
  select_body<256>(K, q, round, b_idx, thr, reach, handled, correct_total, st, hist);
}

// All K-1 rounds in one cooperative launch (single GPU): histogram by every
// CTA -> grid barrier -> select by CTA 0 -> grid barrier -> next round.
__global__ void __launch_bounds__(1024) calib_fused_kernel(const float* __restrict__ conf,
                                                           const uint8_t* __restrict__ correct,
                                                           int K, int64_t N, int q, long long target,
                                                           int32_t* b_idx, float* thr,
                                                           int64_t* reach, int64_t* handled,
                                                           int64_t* correct_total, CalibState* st,
                                                           int32_t* hist) {
  pdl_start();
  extern __shared__ unsigned sh[];
  cg::grid_group grid = cg::this_grid();
#ifdef HS_CALIB_TRACE
  int tr = 0;
#define HS_TR(tag)                                                             \
  if (blockIdx.x == 0 && threadIdx.x == 0 && tr < 64) {                        \
    unsigned long long tt;                                                     \
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(tt));                     \
    g_calib_trace[tr++] = tt;                                                  \
  }
#else
#define HS_TR(tag)
#endif
  int k = -1;
  if (blockIdx.x == 0) {
    const int nw = 3 * ((1 << q) + 2);
    for (int i = threadIdx.x; i < nw; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
      st->A = 0;
      st->tau = target < 0 ? 0 : target;
      st->tau_ap = target < 0 ? 1 : 0;
    }
  }
  grid.sync();
  HS_TR("init");
  for (k = 0; k < K - 1; ++k) {
    hist_body(conf, correct, K, N, q, k, b_idx, hist, sh);
    HS_TR("hist");
    grid.sync();
    HS_TR("sync1");
    if (blockIdx.x == 0) {
      // pull the summed histogram into shared memory once (and re-zero it for
      // the next round), then select from shared memory
      const int words = 3 * ((1 << q) + 2);
      uint4* g4 = reinterpret_cast<uint4*>(hist);
      uint4* s4 = reinterpret_cast<uint4*>(sh);
      for (int i = threadIdx.x; i < words / 4; i += blockDim.x) {
        s4[i] = g4[i];
        g4[i] = make_uint4(0, 0, 0, 0);
      }
      for (int i = (words / 4) * 4 + threadIdx.x; i < words; i += blockDim.x) {
        sh[i] = (unsigned)hist[i];
        hist[i] = 0;
      }
      __syncthreads();
      HS_TR("pulled");
      select_core<1024>(SharedHist{sh, (1 << q) + 2}, K, q, k, b_idx, thr, reach, handled,
                        correct_total, st);
      HS_TR("select");
    }
    grid.sync();
    HS_TR("sync2");
  }
}

// All K-1 rounds on ONE thread-block cluster (validation sets below 2^20):
// every CTA builds a private shared-memory histogram of its samples, the
// cluster barrier publishes them, CTA rank 0 sums the other CTAs' histograms
// through distributed shared memory (DSMEM loads), writes the combined
// histogram once and runs the select; a second cluster barrier releases the
// next round.  No global atomics and no grid-wide barrier.
__global__ void __launch_bounds__(1024, 1) calib_cluster_kernel(const float* __restrict__ conf,
                                                             const uint8_t* __restrict__ correct,
                                                             int K, int64_t N, int q,
                                                             long long target, int32_t* b_idx,
                                                             float* thr, int64_t* reach,
                                                             int64_t* handled,
                                                             int64_t* correct_total,
                                                             CalibState* st, int32_t* hist) {
  pdl_start();
  extern __shared__ unsigned sh[];
  cg::cluster_group cluster = cg::this_cluster();
  const unsigned rank = cluster.block_rank(), ncta = cluster.num_blocks();
  const int nb = (1 << q) + 2;
  if (rank == 0) {
    for (int i = threadIdx.x; i < 3 * nb; i += blockDim.x) hist[i] = 0;
    if (threadIdx.x == 0) {
      st->A = 0;
      st->tau = target < 0 ? 0 : target;
      st->tau_ap = target < 0 ? 1 : 0;
    }
  }
  cluster.sync();
  for (int k = 0; k < K - 1; ++k) {
    hist_local(conf, correct, K, N, q, k, b_idx, sh,
               (int64_t)rank * blockDim.x + threadIdx.x, (int64_t)ncta * blockDim.x);
    cluster.sync();
    // ranks 1.. push their non-empty bins into rank 0's histogram (DSMEM atomics)
    if (rank != 0) {
      unsigned* dst = cluster.map_shared_rank(sh, 0);
      for (int i = threadIdx.x; i < 3 * nb; i += blockDim.x) {
        const unsigned v = sh[i];
        if (v) atomicAdd(dst + i, v);
      }
    }
    cluster.sync();
    if (rank == 0)
      select_core<1024>(SharedHist{sh, nb}, K, q, k, b_idx, thr, reach, handled, correct_total, st);
    cluster.sync();
  }
}

// ---------------------------------------------------------------------------
// Resident variant of the cooperative kernel (default when the samples fit):
// every CTA loads ITS samples once -- the fp32 bins of stages 0..K-2 (int16,
// NaN -> -1) and the K correct bits -- into shared memory, so a round touches
// no per-sample global memory.  One grid barrier per round: the CTAs flush
// their histograms into a rotating set of three global buffers (round k uses
// buffer k % 3 and zeroes buffer (k+1) % 3, which every CTA stopped reading
// two barriers ago), then EVERY CTA pulls the summed histogram and runs the
// same deterministic select, so nobody waits for a broadcast of b_k.  CTA 0
// alone writes the outputs.
//
// The global buffers hold one packed u64 per bin -- count | correct_k << 21 |
// correct_K << 42 (N < 2^21, checked by the launcher) -- so a flush is one
// red.add.u64 per non-empty bin, and the select reads its contiguous bins
// straight from L2 into registers (no shared-memory staging of the histogram).
// ---------------------------------------------------------------------------
struct SelState {            // per-CTA copy of the select state + outputs
  CalibState st;
  int32_t b[16];
  float t[17];
  int64_t reach[17], handled[17], total;
};

constexpr int kPackBits = 21;
constexpr unsigned long long kPackMask = (1ull << kPackBits) - 1;

// select_core's three passes (same arithmetic, same tie rules) on a packed
// global histogram whose bins [lo, lo + n) sit in this thread's registers.
template <int NT, int PMAX, bool SMEM = false>
__device__ __forceinline__ void select_packed(const unsigned long long* __restrict__ g, int K,
                                              int q, int round, SelState* ss, int nsum = 1,
                                              int sum_stride = 0) {
  constexpr int NW = NT / 32;
  static_assert(NW <= 32, "one warp scans the warp totals");
  __shared__ int sh_x[NW], sh_y[NW], sh_z[NW], sh_u[NW];
  __shared__ int sh_tot[2];
  __shared__ int sh_bk;
  __shared__ long long sh_tau, sh_A;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B = 1 << q;
  const int per = (B + 1 + NT - 1) / NT;          // <= PMAX (checked by the launcher)
  const int lo = min(tid * per, B + 1), n = min(per, B + 1 - lo);
  unsigned long long v[PMAX];
#pragma unroll
  for (int i = 0; i < PMAX; ++i) v[i] = i < n ? (SMEM ? g[lo + i + 1] : __ldcg(g + lo + i + 1)) : 0ull;
  unsigned long long v0 = tid == 0 ? (SMEM ? g[0] : __ldcg(g)) : 0ull;   // NaN bin: never accepted
  // multi-GPU: the W ranks' packed histograms (pushed into this rank's peer
  // region) are summed here; packed fields cannot carry (global N < 2^21)
  for (int w = 1; w < nsum; ++w) {
    const unsigned long long* gw = g + (size_t)w * sum_stride;
#pragma unroll
    for (int i = 0; i < PMAX; ++i) v[i] += i < n ? __ldcg(gw + lo + i + 1) : 0ull;
    if (tid == 0) v0 += __ldcg(gw);
  }
#define HS_CNT(x) ((int)((x) & kPackMask))
#define HS_CK(x) ((int)(((x) >> kPackBits) & kPackMask))
#define HS_CKK(x) ((int)((x) >> (2 * kPackBits)))
  // ---- pass 1
  int segH = 0, segCnt = HS_CNT(v0), segK = HS_CKK(v0);
#pragma unroll
  for (int i = 0; i < PMAX; ++i) {
    segH += HS_CK(v[i]) - HS_CKK(v[i]);
    segCnt += HS_CNT(v[i]);
    segK += HS_CKK(v[i]);
  }
  int incl = segH;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int y = __shfl_down_sync(0xFFFFFFFFu, incl, o);
    if (lane + o < 32) incl += y;
  }
  const int wc = __reduce_add_sync(0xFFFFFFFFu, segCnt);
  const int wk = __reduce_add_sync(0xFFFFFFFFu, segK);
  if (lane == 0) {
    sh_x[wid] = incl;
    sh_y[wid] = wc;
    sh_z[wid] = wk;
  }
  __syncthreads();
  if (wid == 0) {
    const int h = lane < NW ? sh_x[lane] : 0;
    int suf = h;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_down_sync(0xFFFFFFFFu, suf, o);
      if (lane + o < 32) suf += y;
    }
    const int tc = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_y[lane] : 0);
    const int tk = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_z[lane] : 0);
    if (lane < NW) sh_u[lane] = suf - h;
    if (lane == 0) {
      sh_tot[0] = tc;
      sh_tot[1] = tk;
      if (round == 0 && ss->st.tau_ap) ss->st.tau = tk;   // AP: tau = correct answers of m_K
      sh_tau = ss->st.tau;
      sh_A = ss->st.A;
    }
  }
  __syncthreads();
  const long long reach_k = sh_tot[0], G = sh_tot[1], tau = sh_tau, A = sh_A;
  // ---- pass 2
  int best = B + 1;
  {
    long long S = (long long)sh_u[wid] + (incl - segH);
#pragma unroll
    for (int i = PMAX - 1; i >= 0; --i) {
      if (i < n) {
        S += HS_CK(v[i]) - HS_CKK(v[i]);
        if (A + G + S >= tau) best = lo + i;
      }
    }
  }
  best = (int)__reduce_min_sync(0xFFFFFFFFu, (unsigned)best);
  if (lane == 0) sh_x[wid] = best;
  __syncthreads();
  if (wid == 0) {
    const unsigned x = lane < NW ? (unsigned)sh_x[lane] : (unsigned)(B + 1);
    const int bk = (int)__reduce_min_sync(0xFFFFFFFFu, x);
    if (lane == 0) sh_bk = bk;
  }
  __syncthreads();
  const int bk = sh_bk;
  // ---- pass 3
  int s_ck = 0, s_cnt = 0, s_bc = HS_CNT(v0), s_bK = HS_CKK(v0);
#pragma unroll
  for (int i = 0; i < PMAX; ++i) {
    if (lo + i >= bk) {              // empty tail slots are zero
      s_ck += HS_CK(v[i]);
      s_cnt += HS_CNT(v[i]);
    } else {
      s_bc += HS_CNT(v[i]);
      s_bK += HS_CKK(v[i]);
    }
  }
#undef HS_CNT
#undef HS_CK
#undef HS_CKK
  s_ck = __reduce_add_sync(0xFFFFFFFFu, s_ck);
  s_cnt = __reduce_add_sync(0xFFFFFFFFu, s_cnt);
  s_bc = __reduce_add_sync(0xFFFFFFFFu, s_bc);
  s_bK = __reduce_add_sync(0xFFFFFFFFu, s_bK);
  if (lane == 0) {
    sh_x[wid] = s_ck;
    sh_y[wid] = s_cnt;
    sh_z[wid] = s_bc;
    sh_u[wid] = s_bK;
  }
  __syncthreads();
  if (wid == 0) {
    const int ck = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_x[lane] : 0);
    const int cnt = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_y[lane] : 0);
    const int bc = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_z[lane] : 0);
    const int bK = __reduce_add_sync(0xFFFFFFFFu, lane < NW ? sh_u[lane] : 0);
    if (lane == 0) {
      long long Anew = A + ck;
      ss->b[round] = bk;
      ss->t[round] = bk <= B ? (float)bk / (float)B : INFINITY;
      ss->reach[round] = reach_k;
      ss->handled[round] = cnt;
      if (round == K - 2) {
        ss->reach[K - 1] = bc;
        ss->handled[K - 1] = bc;
        Anew += bK;
        ss->t[K - 1] = 0.f;
        ss->total = Anew;
      }
      ss->st.A = Anew;
    }
  }
  __syncthreads();
}

constexpr int kResidentThreads = 1024;

// PMAX = bins per thread in the select, ceil((2^q + 1) / 1024): one
// instantiation per range of q keeps the bins in registers.
// Multi-GPU round exchange over peer memory (peer.cu layout): this rank's
// packed histogram of round r (global round index, parity p = r & 1) is pushed
// into slot [p][rank] of every rank's region (CTA c serves ranks c, c + grid,
// ...), each push followed by a system-scope release increment of that rank's
// arrival counter p; every CTA then waits until its own counter p reached
// (r/2 + 1) * W and the select sums the W slots.  A slot of parity p is
// rewritten two rounds later, by a rank that has seen every peer's push of
// the round in between -- pushed after that peer's CTAs finished reading it.
__device__ __forceinline__ void red_release_sys_add(unsigned long long* p, unsigned long long v) {
  asm volatile("red.release.sys.global.add.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}
__device__ __forceinline__ unsigned long long ld_acquire_sys_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void peer_push_wait(const PeerCal& pc, const unsigned long long* hist,
                                               bool hist_smem, int nb, unsigned long long r) {
  const int par = (int)(r & 1), W = pc.world;
  for (int h = blockIdx.x; h < W; h += gridDim.x) {
    unsigned long long* dst = pc.slots[h] + ((size_t)par * W + pc.rank) * nb;
    for (int i = threadIdx.x; i < nb; i += blockDim.x) dst[i] = hist_smem ? hist[i] : __ldcg(hist + i);
    __syncthreads();
    if (threadIdx.x == 0) {
      __threadfence_system();
      red_release_sys_add(pc.arrive[h] + par, 1ull);
    }
  }
  if (threadIdx.x == 0) {
    const unsigned long long want = ((r >> 1) + 1) * (unsigned long long)W;
    const unsigned long long* a = pc.arrive[pc.rank] + par;
    unsigned long long t0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t0));
    while (ld_acquire_sys_u64(a) < want) {
      unsigned long long t;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
      if (t - t0 > 10ull * 1000 * 1000 * 1000) {      // a peer never pushed: give up, flag it
        if (pc.status) atomicOr(pc.status, HS_STATUS_TIMEOUT);
        break;
      }
      __nanosleep(128);
    }
  }
  __syncthreads();
}

template <int PMAX, bool PEER>
__global__ void __launch_bounds__(kResidentThreads, 1) calib_resident_kernel(
    const float* __restrict__ conf, const uint8_t* __restrict__ correct, int K, int64_t N, int q,
    long long target, int32_t* b_idx, float* thr, int64_t* reach, int64_t* handled,
    int64_t* correct_total, CalibState* st_out, unsigned long long* hist3, int per_cta,
    const __grid_constant__ PeerCal pc) {
  pdl_start();
  const unsigned long long rbase = PEER ? *pc.round_ctr : 0ull;   // read before the first grid barrier
#ifdef HS_CALIB_TRACE
  int tr = 0;
#endif
  extern __shared__ __align__(16) unsigned char smraw[];
  cg::grid_group grid = cg::this_grid();
  const int nb = (1 << q) + 2;
  const int hw = 3 * nb;                                   // u32 words of the local histogram
  unsigned* sh = reinterpret_cast<unsigned*>(smraw);        // local histogram (SoA)
  SelState* ss = reinterpret_cast<SelState*>(smraw + (size_t)hw * 4 + 16 - ((size_t)hw * 4) % 16);
  int16_t* sbin = reinterpret_cast<int16_t*>(ss + 1);       // [(K-1) x per_cta]
  uint16_t* sok = reinterpret_cast<uint16_t*>(sbin + (size_t)(K - 1) * per_cta);
  const int tid = threadIdx.x;
  const int64_t r0 = (int64_t)blockIdx.x * per_cta;
  const int m = (int)max((int64_t)0, min((int64_t)per_cta, N - r0));
  // ---- resident samples
  for (int i = tid; i < m; i += blockDim.x) {
    const int64_t r = r0 + i;
    uint16_t ok = 0;
    for (int k = 0; k < K; ++k) ok |= (uint16_t)(__ldg(correct + (int64_t)k * N + r) != 0) << k;
    sok[i] = ok;
    for (int k = 0; k < K - 1; ++k) sbin[(size_t)k * per_cta + i] = (int16_t)bin_of(__ldg(conf + (int64_t)k * N + r), q);
  }
  for (int i = tid; i < hw; i += blockDim.x) sh[i] = 0u;   // the flush re-zeroes it
  if (tid == 0) {
    ss->st.A = 0;
    ss->st.tau = target < 0 ? 0 : target;
    ss->st.tau_ap = target < 0 ? 1 : 0;
  }
  // buffer 0 must be zero for round 0: zeroed here, ordered by the first barrier
  for (int i = blockIdx.x * blockDim.x + tid; i < nb; i += gridDim.x * blockDim.x) hist3[i] = 0ull;
  grid.sync();
  HS_TR("init");
  const int mup = (m + 31) & ~31;
  const bool aggregate = q < 8;      // block-uniform
  // one CTA (small validation sets, e.g. C1): the packed bins stay in shared
  // memory and the round needs no grid barrier and no global atomics
  const bool solo = gridDim.x == 1;
  unsigned long long* spk = reinterpret_cast<unsigned long long*>(
      reinterpret_cast<unsigned char*>(sok + per_cta) + (16 - (reinterpret_cast<uintptr_t>(sok + per_cta) & 15)));
  for (int k = 0; k < K - 1; ++k) {
    unsigned long long* cur = hist3 + (size_t)(k % 3) * nb;
    unsigned long long* nxt = hist3 + (size_t)((k + 1) % 3) * nb;
    for (int i = blockIdx.x * blockDim.x + tid; i < nb; i += gridDim.x * blockDim.x) nxt[i] = 0ull;
    for (int i = tid; i < mup; i += blockDim.x) {
      bool alive = i < m;
      int key = -1;
      bool okk = false, okK = false;
      if (alive) {
        for (int j = 0; j < k; ++j) alive &= sbin[(size_t)j * per_cta + i] < ss->b[j];
        if (alive) {
          const uint16_t ok = sok[i];
          key = sbin[(size_t)k * per_cta + i] + 1;
          okk = (ok >> k) & 1u;
          okK = (ok >> (K - 1)) & 1u;
        }
      }
      if (!aggregate) {            // many bins: lanes rarely share one
        if (key >= 0) {
          atomicAdd(&sh[key], 1u);
          if (okk) atomicAdd(&sh[nb + key], 1u);
          if (okK) atomicAdd(&sh[2 * nb + key], 1u);
        }
        continue;
      }
      // few bins: lanes with the same bin add once, through their leader
      const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
      const unsigned bk = __ballot_sync(0xFFFFFFFFu, okk);
      const unsigned bK = __ballot_sync(0xFFFFFFFFu, okK);
      if (key >= 0 && (tid & 31) == __ffs(peers) - 1) {
        atomicAdd(&sh[key], (unsigned)__popc(peers));
        const unsigned nk = __popc(peers & bk), nK = __popc(peers & bK);
        if (nk) atomicAdd(&sh[nb + key], nk);
        if (nK) atomicAdd(&sh[2 * nb + key], nK);
      }
    }
    __syncthreads();
    HS_TR("local");
    for (int i = tid; i < nb; i += blockDim.x) {
      const unsigned c = sh[i];
      if (solo) {
        const unsigned long long ck = sh[nb + i], cK = sh[2 * nb + i];
        sh[i] = 0u;
        sh[nb + i] = 0u;
        sh[2 * nb + i] = 0u;
        spk[i] = (unsigned long long)c | (ck << kPackBits) | (cK << (2 * kPackBits));
      } else if (c) {       // correct counts are only taken on counted samples
        const unsigned long long ck = sh[nb + i], cK = sh[2 * nb + i];
        sh[i] = 0u;
        sh[nb + i] = 0u;
        sh[2 * nb + i] = 0u;
        atomicAdd(cur + i, (unsigned long long)c | (ck << kPackBits) | (cK << (2 * kPackBits)));
      }
    }
    HS_TR("flush");
    if (solo) {
      __syncthreads();
      if (PEER) {
        const unsigned long long r = rbase + k;
        peer_push_wait(pc, spk, true, nb, r);
        select_packed<kResidentThreads, PMAX>(pc.slots[pc.rank] + (size_t)(r & 1) * pc.world * nb, K, q,
                                              k, ss, pc.world, nb);
      } else {
        select_packed<kResidentThreads, PMAX, true>(spk, K, q, k, ss);
      }
      HS_TR("select");
      continue;
    }
    grid.sync();
    HS_TR("sync");
    if (PEER) {
      const unsigned long long r = rbase + k;
      peer_push_wait(pc, cur, false, nb, r);
      select_packed<kResidentThreads, PMAX>(pc.slots[pc.rank] + (size_t)(r & 1) * pc.world * nb, K, q, k,
                                            ss, pc.world, nb);
    } else {
      // every CTA selects from the summed histogram (identical results)
      select_packed<kResidentThreads, PMAX>(cur, K, q, k, ss);
    }
    HS_TR("select");
  }
  if (PEER && blockIdx.x == 0 && threadIdx.x == 0) *pc.round_ctr = rbase + (unsigned long long)(K - 1);
  if (blockIdx.x == 0) {
    for (int k = tid; k < K; k += blockDim.x) {
      if (k < K - 1) b_idx[k] = ss->b[k];
      thr[k] = ss->t[k];
      reach[k] = ss->reach[k];
      handled[k] = ss->handled[k];
    }
    if (tid == 0) {
      *correct_total = ss->total;
      *st_out = ss->st;            // refinement passes continue from tau (D5)
    }
  }
}

// ---------------------------------------------------------------------------
// Optional refinement passes: re-pick each b_k given the
// current downstream thresholds.  Round k of a pass histograms the samples that
// still reach model k under the current thresholds, with the third channel
// holding the correctness of the DOWNSTREAM cascade (k+1 .. K-1 under the
// current b) instead of correct_K, and accumulates A_k = correct answers given
// before k.  The ordinary select then yields
//   b_k = min{ b : A_k + sum_{bin>=b} correct_k + sum_{bin<b} C_down >= tau }.
// ---------------------------------------------------------------------------
__global__ void calib_refine_begin_kernel(CalibState* st) {
  pdl_start();
  if (threadIdx.x == 0) {
    st->A = 0;
    st->tau_ap = 0;   // tau is fixed by the greedy pass
  }
}

__global__ void __launch_bounds__(512) calib_refine_hist_kernel(const float* __restrict__ conf,
                                                                const uint8_t* __restrict__ correct,
                                                                int K, int64_t N, int q, int k,
                                                                const int32_t* __restrict__ b_idx,
                                                                int32_t* __restrict__ hist,
                                                                CalibState* st) {
  pdl_start();
  extern __shared__ unsigned sh[];
  __shared__ int s_b[16];
  __shared__ unsigned long long s_A;
  const int nb = (1 << q) + 2;
  hist_zero(sh, q);
  if (threadIdx.x < 16) s_b[threadIdx.x] = threadIdx.x < K - 1 ? b_idx[threadIdx.x] : 0;
  if (threadIdx.x == 0) s_A = 0ull;
  __syncthreads();
  unsigned long long myA = 0;
  const int64_t Nup = (N + 31) & ~(int64_t)31;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < Nup;
       r += (int64_t)gridDim.x * blockDim.x) {
    const bool in = r < N;
    int key = -1;
    bool okk = false, okD = false;
    if (in) {
      int j = 0;
      while (j < k && bin_of(__ldg(conf + (int64_t)j * N + r), q) < s_b[j]) ++j;
      if (j < k) {
        myA += __ldg(correct + (int64_t)j * N + r);
      } else {
        int d = k + 1;
        while (d < K - 1 && bin_of(__ldg(conf + (int64_t)d * N + r), q) < s_b[d]) ++d;
        key = bin_of(__ldg(conf + (int64_t)k * N + r), q) + 1;
        okk = __ldg(correct + (int64_t)k * N + r) != 0;
        okD = __ldg(correct + (int64_t)d * N + r) != 0;
      }
    }
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
    const unsigned bk = __ballot_sync(0xFFFFFFFFu, okk);
    const unsigned bD = __ballot_sync(0xFFFFFFFFu, okD);
    if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) {
      atomicAdd(&sh[key], (unsigned)__popc(peers));
      const unsigned nk = __popc(peers & bk), nD = __popc(peers & bD);
      if (nk) atomicAdd(&sh[nb + key], nk);
      if (nD) atomicAdd(&sh[2 * nb + key], nD);
    }
  }
  myA = warp_sum(myA);
  if ((threadIdx.x & 31) == 0 && myA) atomicAdd(&s_A, myA);
  __syncthreads();
  hist_flush(sh, q, hist);
  if (threadIdx.x == 0 && s_A) atomicAdd(reinterpret_cast<unsigned long long*>(&st->A), s_A);
}

// Final replay under the chosen thresholds: reach / handled per model and the
// cascade's correct count (after refinement passes).
__global__ void calib_replay_zero_kernel(int K, int64_t* reach, int64_t* handled,
                                         int64_t* correct_total) {
  pdl_start();
  for (int k = threadIdx.x; k < K; k += blockDim.x) {
    reach[k] = 0;
    handled[k] = 0;
  }
  if (threadIdx.x == 0) *correct_total = 0;
}

__global__ void __launch_bounds__(512) calib_replay_kernel(const float* __restrict__ conf,
                                                           const uint8_t* __restrict__ correct,
                                                           int K, int64_t N, int q,
                                                           const int32_t* __restrict__ b_idx,
                                                           int64_t* reach, int64_t* handled,
                                                           int64_t* correct_total) {
  pdl_start();
  __shared__ int s_b[16];
  __shared__ unsigned long long s_reach[17], s_hand[17], s_ok;
  if (threadIdx.x < 17) {
    s_reach[threadIdx.x] = 0;
    s_hand[threadIdx.x] = 0;
  }
  if (threadIdx.x < 16) s_b[threadIdx.x] = threadIdx.x < K - 1 ? b_idx[threadIdx.x] : 0;
  if (threadIdx.x == 0) s_ok = 0;
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < N;
       r += (int64_t)gridDim.x * blockDim.x) {
    int j = 0;
    while (j < K - 1 && bin_of(__ldg(conf + (int64_t)j * N + r), q) < s_b[j]) ++j;
    for (int i = 0; i <= j; ++i) atomicAdd(&s_reach[i], 1ull);
    atomicAdd(&s_hand[j], 1ull);
    if (__ldg(correct + (int64_t)j * N + r)) atomicAdd(&s_ok, 1ull);
  }
  __syncthreads();
  if (threadIdx.x < K) {
    if (s_reach[threadIdx.x]) atomicAdd(reinterpret_cast<unsigned long long*>(&reach[threadIdx.x]), s_reach[threadIdx.x]);
    if (s_hand[threadIdx.x]) atomicAdd(reinterpret_cast<unsigned long long*>(&handled[threadIdx.x]), s_hand[threadIdx.x]);
  }
  if (threadIdx.x == 0 && s_ok) atomicAdd(reinterpret_cast<unsigned long long*>(correct_total), s_ok);
}

}  // namespace

size_t calib_hist_bytes(int q) { return (size_t)3 * ((1u << q) + 2) * sizeof(int32_t); }
size_t calib_ws_bytes(int K, int q) {
  (void)K;
  return sizeof(CalibState) + 3 * calib_hist_bytes(q);   // 3 rotating buffers (resident kernel)
}

static int32_t* hist_of(void* ws) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + sizeof(CalibState));
}

cudaError_t launch_calib_init(void* ws, int q, long long target, cudaStream_t s) {
  return launch_pdl(calib_init_kernel, dim3(1), dim3(1024), 0, s, reinterpret_cast<CalibState*>(ws),
                    hist_of(ws), 3 * ((1 << q) + 2), target);
}

cudaError_t launch_calib_hist(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                              int round, const int32_t* b_idx, int32_t* hist, cudaStream_t s) {
  const size_t smem = (size_t)3 * ((1 << q) + 2) * sizeof(unsigned);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(calib_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(3 * ((1 << 14) + 2) * sizeof(unsigned)));
    attr = true;
  }
  int64_t grid = (N + 512 * 8 - 1) / (512 * 8);
  const int64_t cap = (int64_t)num_sms() * 2;
  if (grid > cap) grid = cap;
  if (grid < 1) grid = 1;
  return launch_pdl(calib_hist_kernel, dim3((int)grid), dim3(512), smem, s, conf, correct, K, N, q,
                    round, b_idx, hist);
}

static cudaError_t launch_calib_resident(const float* conf, const uint8_t* correct, int K,
                                        int64_t N, int q, long long target, int32_t* b_idx,
                                        float* thr, int64_t* reach, int64_t* handled,
                                        int64_t* correct_total, void* ws, cudaStream_t s,
                                        bool* launched, const PeerCal* peer = nullptr) {
  *launched = false;
  const size_t hbytes = (size_t)3 * ((1 << q) + 2) * sizeof(unsigned);
  const size_t head = hbytes + 16 - hbytes % 16 + sizeof(SelState);
  const size_t cap = 220 * 1024;
  int grid = (int)((N + 4095) / 4096);
  if (grid > num_sms()) grid = num_sms();
  if (grid < 1) grid = 1;
  const int64_t per = (N + grid - 1) / grid;
  size_t smem = head + (size_t)per * (2 * (size_t)(K - 1) + 2) + 16;
  if (grid == 1) smem += (size_t)((1 << q) + 2) * sizeof(unsigned long long) + 16;   // packed bins (solo)
  // packed u64 bins need N < 2^21; K <= 16 correct bits per sample
  // (multi-GPU: the packed fields hold sums over every rank's shard; shards of
  // equal size assumed, N * world < 2^21)
  const int64_t n_glob = N * (peer ? (int64_t)peer->world : 1);
  if (K > 16 || n_glob >= (int64_t(1) << kPackBits) || q > 14 || smem > cap) return cudaSuccess;
  const int pm = q <= 9 ? 1 : q <= 11 ? 3 : q == 12 ? 5 : q == 13 ? 9 : 17;
  using Kern = void (*)(const float*, const uint8_t*, int, int64_t, int, long long, int32_t*, float*,
                        int64_t*, int64_t*, int64_t*, CalibState*, unsigned long long*, int, PeerCal);
  static const Kern kerns[2][5] = {
      {calib_resident_kernel<1, false>, calib_resident_kernel<3, false>, calib_resident_kernel<5, false>,
       calib_resident_kernel<9, false>, calib_resident_kernel<17, false>},
      {calib_resident_kernel<1, true>, calib_resident_kernel<3, true>, calib_resident_kernel<5, true>,
       calib_resident_kernel<9, true>, calib_resident_kernel<17, true>}};
  const int slot = pm == 1 ? 0 : pm == 3 ? 1 : pm == 5 ? 2 : pm == 9 ? 3 : 4;
  const int pe = peer ? 1 : 0;
  Kern kern = kerns[pe][slot];
  static bool attr[2][5] = {};
  if (!attr[pe][slot]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)cap);
    attr[pe][slot] = true;
  }
  PeerCal pc{};
  if (peer) pc = *peer;
  int per_sm = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kResidentThreads, smem);
  if (per_sm < 1 || grid > per_sm * num_sms()) return cudaSuccess;
  // 3 x (B+2) u64 fit in the 3 x 3 x (B+2) u32 the workspace reserves
  unsigned long long* hist3 = reinterpret_cast<unsigned long long*>(hist_of(ws));
  CalibState* st = reinterpret_cast<CalibState*>(ws);
  int per_cta = (int)per;
  void* args[] = {(void*)&conf, (void*)&correct, (void*)&K, (void*)&N, (void*)&q, (void*)&target,
                  (void*)&b_idx, (void*)&thr, (void*)&reach, (void*)&handled,
                  (void*)&correct_total, (void*)&st, (void*)&hist3, (void*)&per_cta, (void*)&pc};
  // cooperative (grid barriers) + programmatic dependent launch: the CTAs are
  // placed as the previous kernel's CTAs retire and wait in griddepcontrol.wait
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kResidentThreads);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  cudaError_t e = cudaLaunchKernelExC(&cfg, (const void*)kern, args);
  count_launch();
  *launched = true;
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_calib_fused(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                               long long target, int32_t* b_idx, float* thr, int64_t* reach,
                               int64_t* handled, int64_t* correct_total, void* ws,
                               cudaStream_t s) {
  if (!getenv("HS_CALIB_NORESIDENT")) {
    bool launched = false;
    const cudaError_t e = launch_calib_resident(conf, correct, K, N, q, target, b_idx, thr, reach,
                                                handled, correct_total, ws, s, &launched);
    if (launched || e != cudaSuccess) return e;
  }
  const size_t smem = (size_t)3 * ((1 << q) + 2) * sizeof(unsigned);
  static int max_blocks = -1;
  if (max_blocks < 0) {
    cudaFuncSetAttribute(calib_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(3 * ((1 << 14) + 2) * sizeof(unsigned)));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, calib_fused_kernel, 1024,
                                                  3 * ((1 << 14) + 2) * sizeof(unsigned));
    max_blocks = per_sm > 0 ? per_sm * num_sms() : 0;
  }
  // ~4K samples per CTA: enough parallelism for the histogram pass while
  // keeping the flush (global atomics on the hot bins near c = 1) small
  int grid = (int)((N + 4095) / 4096);
  if (grid > num_sms()) grid = num_sms();
  if (grid > max_blocks) grid = max_blocks;
  if (grid < 1) grid = 1;
  CalibState* st = reinterpret_cast<CalibState*>(ws);
  int32_t* hist = hist_of(ws);
  void* args[] = {(void*)&conf, (void*)&correct, (void*)&K, (void*)&N, (void*)&q, (void*)&target,
                  (void*)&b_idx, (void*)&thr, (void*)&reach, (void*)&handled,
                  (void*)&correct_total, (void*)&st, (void*)&hist};
  cudaError_t e = cudaLaunchCooperativeKernel((void*)calib_fused_kernel, dim3(grid), dim3(1024),
                                              args, smem, s);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// Multi-GPU calibration over peer memory: the resident kernel only (the
// samples of this rank's shard must fit its shared memory, N * world < 2^21);
// returns cudaErrorNotSupported when it cannot be used.
cudaError_t launch_calib_peer(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                              long long target, int32_t* b_idx, float* thr, int64_t* reach,
                              int64_t* handled, int64_t* correct_total, void* ws, const PeerCal& pc,
                              cudaStream_t s) {
  bool launched = false;
  const cudaError_t e = launch_calib_resident(conf, correct, K, N, q, target, b_idx, thr, reach, handled,
                                              correct_total, ws, s, &launched, &pc);
  if (e != cudaSuccess) return e;
  return launched ? cudaSuccess : cudaErrorNotSupported;
}

// Building blocks of the refinement for a sharded validation set (the caller
// sums the histogram + A, and the replay counts, across ranks in between).
cudaError_t launch_calib_refine_round(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                                      int k, const int32_t* b_idx, void* ws, bool zero_hist, cudaStream_t s) {
  CalibState* st = reinterpret_cast<CalibState*>(ws);
  int32_t* hist = hist_of(ws);
  const size_t smem = (size_t)3 * ((1 << q) + 2) * sizeof(unsigned);
  static const bool attr = [] {
    cudaFuncSetAttribute(calib_refine_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(3 * ((1 << 14) + 2) * sizeof(unsigned)));
    return true;
  }();
  (void)attr;
  int64_t grid = (N + 4095) / 4096;
  if (grid > num_sms()) grid = num_sms();
  if (grid < 1) grid = 1;
  cudaError_t e = zero_hist ? cudaMemsetAsync(hist, 0, calib_hist_bytes(q), s) : cudaSuccess;
  if (e == cudaSuccess) e = launch_pdl(calib_refine_begin_kernel, dim3(1), dim3(32), 0, s, st);
  if (e == cudaSuccess && N > 0)
    e = launch_pdl(calib_refine_hist_kernel, dim3((int)grid), dim3(512), smem, s, conf, correct, K, N, q, k,
                   b_idx, hist, st);
  return e;
}

cudaError_t launch_calib_replay(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                                const int32_t* b_idx, int64_t* reach, int64_t* handled, int64_t* correct_total,
                                cudaStream_t s) {
  int64_t grid = (N + 4095) / 4096;
  if (grid > num_sms()) grid = num_sms();
  if (grid < 1) grid = 1;
  cudaError_t e = launch_pdl(calib_replay_zero_kernel, dim3(1), dim3(32), 0, s, K, reach, handled, correct_total);
  if (e == cudaSuccess && N > 0)
    e = launch_pdl(calib_replay_kernel, dim3((int)grid), dim3(512), 0, s, conf, correct, K, N, q, b_idx, reach,
                   handled, correct_total);
  return e;
}

cudaError_t launch_calib_refine(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                                int passes, int32_t* b_idx, float* thr, int64_t* reach,
                                int64_t* handled, int64_t* correct_total, void* ws,
                                cudaStream_t s) {
  CalibState* st = reinterpret_cast<CalibState*>(ws);
  int32_t* hist = hist_of(ws);
  const size_t smem = (size_t)3 * ((1 << q) + 2) * sizeof(unsigned);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(calib_refine_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(3 * ((1 << 14) + 2) * sizeof(unsigned)));
    attr = true;
  }
  int64_t grid = (N + 4095) / 4096;
  if (grid > num_sms()) grid = num_sms();
  if (grid < 1) grid = 1;
  // the greedy kernels leave the histogram buffers in an unspecified state
  cudaError_t e = passes > 0 ? cudaMemsetAsync(hist, 0, calib_hist_bytes(q), s) : cudaSuccess;
  for (int p = 0; p < passes && e == cudaSuccess; ++p) {
    for (int k = 0; k < K - 1 && e == cudaSuccess; ++k) {
      e = launch_pdl(calib_refine_begin_kernel, dim3(1), dim3(32), 0, s, st);
      if (e == cudaSuccess)
        e = launch_pdl(calib_refine_hist_kernel, dim3((int)grid), dim3(512), smem, s, conf, correct,
                       K, N, q, k, (const int32_t*)b_idx, hist, st);
      if (e == cudaSuccess)
        e = launch_calib_select(K, q, k, b_idx, thr, reach, handled, correct_total, ws, s);
    }
  }
  if (e == cudaSuccess)
    e = launch_pdl(calib_replay_zero_kernel, dim3(1), dim3(32), 0, s, K, reach, handled, correct_total);
  if (e == cudaSuccess)
    e = launch_pdl(calib_replay_kernel, dim3((int)grid), dim3(512), 0, s, conf, correct, K, N, q,
                   (const int32_t*)b_idx, reach, handled, correct_total);
  return e;
}

constexpr int kCalibCluster = 8;

cudaError_t launch_calib_cluster(const float* conf, const uint8_t* correct, int K, int64_t N,
                                 int q, long long target, int32_t* b_idx, float* thr,
                                 int64_t* reach, int64_t* handled, int64_t* correct_total,
                                 void* ws, cudaStream_t s) {
  const size_t smem = (size_t)3 * ((1 << q) + 2) * sizeof(unsigned);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(calib_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(3 * ((1 << 14) + 2) * sizeof(unsigned)));
    attr = true;
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(kCalibCluster);
  cfg.blockDim = dim3(1024);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = kCalibCluster;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  CalibState* st = reinterpret_cast<CalibState*>(ws);
  int32_t* hist = hist_of(ws);
  cudaError_t e = cudaLaunchKernelEx(&cfg, calib_cluster_kernel, conf, correct, K, N, q, target,
                                     b_idx, thr, reach, handled, correct_total, st, hist);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

cudaError_t launch_calib_select(int K, int q, int round, int32_t* b_idx, float* thr,
                                int64_t* reach, int64_t* handled, int64_t* correct_total,
                                void* ws, cudaStream_t s) {
  return launch_pdl(calib_select_kernel, dim3(1), dim3(256), 0, s, K, q, round, b_idx, thr, reach,
                    handled, correct_total, reinterpret_cast<CalibState*>(ws), hist_of(ws));
}

}  // namespace hs

#ifdef HS_CALIB_TRACE
// experiment builds only: phase timestamps of the last fused calibration launch
extern "C" int hs_debug_calib_trace(unsigned long long* out) {
  return (int)cudaMemcpyFromSymbol(out, hs::g_calib_trace, sizeof(unsigned long long) * 64);
}
#endif
