// calib.cu -- K5 (calibration histogram) and K6 (threshold select).
//
// Offline Accuracy-Preserving threshold calibration (Alg. 1 and
// the AP mode; exact deterministic sweep of DESIGN.md reading G8): thresholds
// live on a 2^q grid, bin(c) = min(B, floor(c * B)) (exact in fp32, so
// bin(c) >= b  <=>  c >= b/B), NaN confidences never accepted.
// Round k (one model) over the validation samples still alive:
//   K5: one pass builds a shared-memory-privatised histogram over bin(c_k) of
//       (count, correct_k, correct_K), packed as ONE 64-bit shared atomic per
//       sample (3 x 21-bit fields), warp-aggregated with __match_any_sync for
//       the skewed bins near c = 1, flushed with global int32 atomics.
//   K6: one CTA: suffix scan over the B+2 bins and
//       b_k = min{ b : A + G + S(b) >= tau } (S is not monotone: every b is
//       examined), then A += committed correct answers; reach/handled counts.
// Histograms are integers, so a request-sharded calibration sums them across
// GPUs (all-reduce) and every rank selects the same b_k.
#include <cooperative_groups.h>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace cg = cooperative_groups;

namespace {

__device__ __forceinline__ int bin_of(float c, int q) {
  if (c != c) return -1;
  const float B = (float)(1 << q);
  float f = floorf(c * B);          // exact: c * 2^q
  f = fminf(fmaxf(f, 0.f), B);
  return (int)f;
}

__global__ void calib_init_kernel(CalibState* st, int32_t* hist, int nwords, long long target) {
  for (int i = threadIdx.x; i < nwords; i += blockDim.x) hist[i] = 0;
  if (threadIdx.x == 0) {
    st->A = 0;
    st->tau = target < 0 ? 0 : target;
    st->tau_ap = target < 0 ? 1 : 0;
  }
}

// hist layout: int32 [3][B+2]; index 0 = NaN bin (never accepted), index b+1 = bin b.
// One CTA's share (grid-stride) of round `round`, added into the global histogram.
__device__ __forceinline__ void hist_body(const float* __restrict__ conf,
                                          const uint8_t* __restrict__ correct, int K, int64_t N,
                                          int q, int round, const int32_t* b_idx,
                                          int32_t* __restrict__ hist, unsigned long long* sh) {
  const int nb = (1 << q) + 2;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) sh[i] = 0ull;
  int bprev[16];
#pragma unroll
  for (int j = 0; j < 16; ++j) bprev[j] = (j < round) ? b_idx[j] : 0;
  __syncthreads();

  const uint8_t* ck = correct + (int64_t)round * N;
  const uint8_t* cK = correct + (int64_t)(K - 1) * N;
  const float* ckconf = conf + (int64_t)round * N;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  // loop bound is warp-uniform so __match_any_sync sees full warps
  const int64_t Nup = (N + 31) & ~(int64_t)31;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < Nup; r += stride) {
    bool alive = r < N;
    if (alive) {
#pragma unroll
      for (int j = 0; j < 16; ++j)
        if (j < round) alive = alive && (bin_of(conf[(int64_t)j * N + r], q) < bprev[j]);
    }
    int key = -1;                      // -1: not counted
    bool okk = false, okK = false;
    if (alive) {
      key = bin_of(ckconf[r], q) + 1;
      okk = ck[r] != 0;
      okK = cK[r] != 0;
    }
    // warp aggregation: lanes with the same bin add once, through their leader
    const unsigned peers = __match_any_sync(0xFFFFFFFFu, key);
    const unsigned bk = __ballot_sync(0xFFFFFFFFu, okk);
    const unsigned bK = __ballot_sync(0xFFFFFFFFu, okK);
    if (key >= 0 && (threadIdx.x & 31) == __ffs(peers) - 1) {
      const unsigned long long tot = (unsigned long long)__popc(peers) |
                                     ((unsigned long long)__popc(peers & bk) << 21) |
                                     ((unsigned long long)__popc(peers & bK) << 42);
      atomicAdd(&sh[key], tot);
    }
  }
  __syncthreads();
  constexpr unsigned long long F = (1ull << 21) - 1;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) {
    const unsigned long long v = sh[i];
    if (v) {
      atomicAdd(&hist[i], (int32_t)(v & F));
      atomicAdd(&hist[nb + i], (int32_t)((v >> 21) & F));
      atomicAdd(&hist[2 * nb + i], (int32_t)((v >> 42) & F));
    }
  }
}

__global__ void __launch_bounds__(512) calib_hist_kernel(const float* __restrict__ conf,
                                                         const uint8_t* __restrict__ correct,
                                                         int K, int64_t N, int q, int round,
                                                         const int32_t* __restrict__ b_idx,
                                                         int32_t* __restrict__ hist) {
  extern __shared__ unsigned long long sh[];
  hist_body(conf, correct, K, N, q, round, b_idx, hist, sh);
}

// One CTA of NT threads.  Each thread owns a contiguous segment of bins
// 0..B (hist index b+1); suffix sums come from a block scan of segment totals.
template <int NT>
__device__ __forceinline__ void select_body(int K, int q, int round, int32_t* b_idx, float* thr,
                                            int64_t* reach, int64_t* handled,
                                            int64_t* correct_total, CalibState* st,
                                            int32_t* hist) {
  constexpr int NW = NT / 32;
  __shared__ long long sh_w[NW];
  __shared__ long long sh_tot[3];
  __shared__ int sh_b;
  __shared__ unsigned long long sh_sum_ck, sh_sum_cnt, sh_below_cnt, sh_below_cK;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int B = 1 << q, nb = B + 2;
  const int32_t* cnt = hist;
  const int32_t* ckh = hist + nb;
  const int32_t* cKh = hist + 2 * nb;

  // ---- totals over all alive samples (incl. the NaN bin): reach_k, G
  long long tc = 0, tK = 0;
  for (int i = tid; i < nb; i += NT) {
    tc += cnt[i];
    tK += cKh[i];
  }
  tc = warp_sum(tc);
  tK = warp_sum(tK);
  if (tid == 0) {
    sh_tot[0] = 0;
    sh_tot[1] = 0;
    sh_b = B + 1;
    sh_sum_ck = sh_sum_cnt = sh_below_cnt = sh_below_cK = 0ull;
  }
  __syncthreads();
  if (lane == 0) {
    atomicAdd((unsigned long long*)&sh_tot[0], (unsigned long long)tc);
    atomicAdd((unsigned long long*)&sh_tot[1], (unsigned long long)tK);
  }
  __syncthreads();
  const long long reach_k = sh_tot[0];
  const long long G = sh_tot[1];
  if (round == 0 && st->tau_ap) {
    if (tid == 0) st->tau = G;      // AP: tau = correct answers of m_K (everything alive)
    __syncthreads();
  }
  const long long tau = st->tau;
  const long long A = st->A;

  // ---- segment of bins [lo, hi) in 0..B, H[b] = ck - cK of bin b
  const int per = (B + 1 + NT - 1) / NT;
  const int lo = min(tid * per, B + 1), hi = min(lo + per, B + 1);
  long long seg = 0;
  for (int b = lo; b < hi; ++b) seg += (long long)ckh[b + 1] - (long long)cKh[b + 1];
  // block exclusive suffix sum of seg (sum over threads with larger tid)
  long long incl = seg;   // inclusive suffix within warp
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const long long y = __shfl_down_sync(0xFFFFFFFFu, incl, o);
    if (lane + o < 32) incl += y;
  }
  if (lane == 0) sh_w[wid] = incl;   // warp total
  __syncthreads();
  long long after_warp = 0;
  for (int v = wid + 1; v < NW; ++v) after_warp += sh_w[v];
  long long suffix = after_warp + (incl - seg);   // sum of H over bins >= hi
  // ---- smallest feasible b in this segment (scan downward keeps S(b) incremental)
  int best = B + 1;
  {
    long long S = suffix;
    for (int b = hi - 1; b >= lo; --b) {
      S += (long long)ckh[b + 1] - (long long)cKh[b + 1];
      if (A + G + S >= tau) best = b;
    }
  }
  atomicMin(&sh_b, best);
  __syncthreads();
  const int bk = sh_b;   // b = B+1 (defer all) is feasible by induction: A + G >= tau
  // ---- commit: A += sum_{bin >= bk} ck ; handled = sum_{bin >= bk} cnt ;
  //      survivors (bin < bk, incl. NaN) for the final stage
  unsigned long long s_ck = 0, s_cnt = 0, s_bc = 0, s_bK = 0;
  for (int i = tid; i < nb; i += NT) {
    const int b = i - 1;   // -1 = NaN bin
    if (b >= bk) {
      s_ck += (unsigned long long)ckh[i];
      s_cnt += (unsigned long long)cnt[i];
    } else {
      s_bc += (unsigned long long)cnt[i];
      s_bK += (unsigned long long)cKh[i];
    }
  }
  s_ck = warp_sum(s_ck);
  s_cnt = warp_sum(s_cnt);
  s_bc = warp_sum(s_bc);
  s_bK = warp_sum(s_bK);
  if (lane == 0) {
    atomicAdd(&sh_sum_ck, s_ck);
    atomicAdd(&sh_sum_cnt, s_cnt);
    atomicAdd(&sh_below_cnt, s_bc);
    atomicAdd(&sh_below_cK, s_bK);
  }
  __syncthreads();
  if (tid == 0) {
    long long Anew = A + (long long)sh_sum_ck;
    b_idx[round] = bk;
    thr[round] = bk <= B ? (float)bk / (float)B : INFINITY;
    reach[round] = reach_k;
    handled[round] = (long long)sh_sum_cnt;
    if (round == K - 2) {
      reach[K - 1] = (long long)sh_below_cnt;
      handled[K - 1] = (long long)sh_below_cnt;
      Anew += (long long)sh_below_cK;
      thr[K - 1] = 0.f;
      *correct_total = Anew;
    }
    st->A = Anew;
  }
  __syncthreads();
  for (int i = tid; i < 3 * nb; i += NT) hist[i] = 0;
}

__global__ void __launch_bounds__(1024) calib_select_kernel(int K, int q, int round,
                                                            int32_t* b_idx, float* thr,
                                                            int64_t* reach, int64_t* handled,
                                                            int64_t* correct_total,
                                                            CalibState* st, int32_t* hist) {
  select_body<1024>(K, q, round, b_idx, thr, reach, handled, correct_total, st, hist);
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
  extern __shared__ unsigned long long sh[];
  cg::grid_group grid = cg::this_grid();
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
  for (int k = 0; k < K - 1; ++k) {
    hist_body(conf, correct, K, N, q, k, b_idx, hist, sh);
    grid.sync();
    if (blockIdx.x == 0) select_body<1024>(K, q, k, b_idx, thr, reach, handled, correct_total, st, hist);
    grid.sync();
  }
}

}  // namespace

size_t calib_hist_bytes(int q) { return (size_t)3 * ((1u << q) + 2) * sizeof(int32_t); }
size_t calib_ws_bytes(int K, int q) {
  (void)K;
  return sizeof(CalibState) + calib_hist_bytes(q);
}

static int32_t* hist_of(void* ws) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + sizeof(CalibState));
}

cudaError_t launch_calib_init(void* ws, int q, long long target, cudaStream_t s) {
  calib_init_kernel<<<1, 1024, 0, s>>>(reinterpret_cast<CalibState*>(ws), hist_of(ws),
                                       3 * ((1 << q) + 2), target);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_calib_hist(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                              int round, const int32_t* b_idx, int32_t* hist, cudaStream_t s) {
  const size_t smem = (size_t)((1 << q) + 2) * sizeof(unsigned long long);
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(calib_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(((1 << 14) + 2) * sizeof(unsigned long long)));
    attr = true;
  }
  // every CTA sees < 2^21 samples per bin field
  int64_t grid = (N + 512 * 8 - 1) / (512 * 8);
  const int64_t cap = (int64_t)num_sms() * 2;
  if (grid > cap) grid = cap;
  const int64_t min_grid = (N >> 20) + 1;
  if (grid < min_grid) grid = min_grid;
  if (grid < 1) grid = 1;
  calib_hist_kernel<<<(int)grid, 512, smem, s>>>(conf, correct, K, N, q, round, b_idx, hist);
  count_launch();
  return cudaGetLastError();
}

cudaError_t launch_calib_fused(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                               long long target, int32_t* b_idx, float* thr, int64_t* reach,
                               int64_t* handled, int64_t* correct_total, void* ws,
                               cudaStream_t s) {
  const size_t smem = (size_t)((1 << q) + 2) * sizeof(unsigned long long);
  static int max_blocks = -1;
  if (max_blocks < 0) {
    cudaFuncSetAttribute(calib_fused_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(((1 << 14) + 2) * sizeof(unsigned long long)));
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, calib_fused_kernel, 1024,
                                                  ((1 << 14) + 2) * sizeof(unsigned long long));
    max_blocks = per_sm > 0 ? per_sm * num_sms() : 0;
  }
  int grid = (int)((N + 1023) / 1024);
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

cudaError_t launch_calib_select(int K, int q, int round, int32_t* b_idx, float* thr,
                                int64_t* reach, int64_t* handled, int64_t* correct_total,
                                void* ws, cudaStream_t s) {
  calib_select_kernel<<<1, 1024, 0, s>>>(K, q, round, b_idx, thr, reach, handled, correct_total,
                                         reinterpret_cast<CalibState*>(ws), hist_of(ws));
  count_launch();
  return cudaGetLastError();
}

}  // namespace hs
