// graph.cu -- NEXT-4: the threshold performance graph of
// Alg. 1 -- replay of many threshold vectors on the validation set,
// its Pareto frontier, and the AP / EO operating points.
//
// Alg. 1 line 4 evaluates a threshold set k by "Compute a on D_v and
// e = sum_i rho_i e_i": the cascade statement replayed on
// every validation sample.  Here every threshold vector is a point of the D5
// grid (b_k in 0..B+1, t_k = b_k / B, B+1 = defer all), so the replay works on
// integer bins: bin(c) >= b_k <=> c >= t_k (reading G10).  rho_i is the reach
// count (G14); energy = sum_k reach_k * w_k with integer weights (G23),
// so every output is an exact integer and the frontier / picks are exact.
//
// K9a replay_prep_kernel: conf -> per-stage int32 bins (SoA, NaN -> -1) and a
//     per-sample correct-bit word; each model's correct count.
// K9b replay_kernel: one thread per threshold vector (given, or digit-decoded
//     from the exhaustive grid index), the samples streamed through shared
//     memory in tiles (every warp reads the same sample: broadcast LDS.128);
//     per sample: K-1 compares -> answering stage (predicated select chain),
//     correct += bit, energy += cumulative weight of the stage (smem table).
//     ALU-bound: ~15 issue slots per (vector, sample).
// K9b' replay_hist_kernel / replay_finish_kernel (the exhaustive grid, B+2 <= 48):
//     vectors sharing the prefix (b_0..b_{K-3}) see the same requests reach
//     model K-2, so per prefix ONE walk over the samples builds a histogram of
//     bin_{K-2} (count, correct_{K-2}, correct_{K-1} packed in a u64, private
//     per thread in shared memory, [bin][thread] so lanes never conflict) plus
//     the correct / energy of the requests answered earlier; the B+2 vectors
//     of the prefix then follow from prefix sums over the histogram (the
//     "joint-histogram prefix table" of SURVEY 8(f) NEXT-4).  (B+2)x fewer
//     sample visits than the direct replay; samples split over CTAs, partial
//     histograms summed with integer atomics (exact).
// K9c graph_*: per correct count c the least energy (64-bit atomicMin) and the
//     lowest vector index achieving it; one CTA then sweeps c downwards
//     (suffix minimum), compacts the Pareto points in ascending c and picks
//     AP (first point with c >= tau) and EO (largest second divided difference
//     of e(c) among interior points with c >= floor, ties to the lowest e).
#include <climits>
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace {

constexpr int kReplayThreads = 256;
// samples per shared-memory tile: (K-1) bins + one bit word per sample, <= 40 KB
__host__ __device__ constexpr int replay_tile(int km1) { return km1 <= 4 ? 2048 : 1024; }
__host__ __device__ constexpr int hist_tile(int) { return 1024; }
constexpr int kFrontThreads = 1024;
constexpr int kFrontTE = 4;                               // counts per thread per tile
constexpr int kFrontTile = kFrontThreads * kFrontTE;

__device__ __forceinline__ int32_t bin_of(float c, int q) {
  if (c != c) return -1;                                  // NaN: never accepted (G20)
  const float f = floorf(c * (float)(1 << q));            // exact: c * 2^q
  const int B = 1 << q;
  return f <= 0.f ? 0 : (f >= (float)B ? B : (int32_t)f);
}

// bins[k * Np + r] (k < K-1), bits[r] (bit k = correct_k), model_correct[k] += ...
__global__ void __launch_bounds__(256) replay_prep_kernel(const float* __restrict__ conf,
                                                          const uint8_t* __restrict__ correct,
                                                          int K, int64_t N, int64_t Np, int q,
                                                          int32_t* bins, uint32_t* bits,
                                                          unsigned long long* model_correct) {
  pdl_start();
  __shared__ unsigned int cnt[32];
  if (threadIdx.x < 32) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < Np;
       r += (int64_t)gridDim.x * blockDim.x) {
    uint32_t w = 0;
    if (r < N) {
      for (int k = 0; k < K; ++k) {
        const uint32_t ok = __ldg(correct + (int64_t)k * N + r) != 0;
        w |= ok << k;
        const unsigned m = __ballot_sync(__activemask(), ok);
        if ((threadIdx.x & 31) == (__ffs(__activemask()) - 1)) atomicAdd(&cnt[k], (unsigned)__popc(m));
      }
      for (int k = 0; k < K - 1; ++k) bins[(int64_t)k * Np + r] = bin_of(__ldg(conf + (int64_t)k * N + r), q);
    } else {
      for (int k = 0; k < K - 1; ++k) bins[(int64_t)k * Np + r] = -1;
    }
    bits[r] = w;
  }
  __syncthreads();
  if (model_correct && threadIdx.x < K && cnt[threadIdx.x])
    atomicAdd(model_correct + threadIdx.x, (unsigned long long)cnt[threadIdx.x]);
}

__global__ void replay_zero_kernel(unsigned long long* model_correct, int K) {
  pdl_start();
  if (threadIdx.x < K) model_correct[threadIdx.x] = 0ull;
}

// KM1 = K-1 compares (compile-time), REACH: per-stage reach counts too
template <int KM1, bool REACH>
__global__ void __launch_bounds__(kReplayThreads) replay_kernel(
    const int32_t* __restrict__ bins, const uint32_t* __restrict__ bits, int64_t N, int64_t Np,
    int q, const int32_t* __restrict__ bvecs, int64_t S, const __grid_constant__ ReplayWeights cw, int64_t* out_c,
    int64_t* out_e, int64_t* out_reach) {
  pdl_start();
  constexpr int K = KM1 + 1;
  constexpr int kReplayTile = replay_tile(KM1);
  __shared__ __align__(16) int32_t sb[KM1][kReplayTile];
  __shared__ __align__(16) uint32_t sk[kReplayTile];
  __shared__ unsigned long long scw[K];
#pragma unroll
  for (int k = 0; k < K; ++k)            // static indices: the parameter stays in the constant bank
    if (threadIdx.x == k) scw[k] = cw.cum[k];
  const int64_t s = (int64_t)blockIdx.x * kReplayThreads + threadIdx.x;
  const bool valid = s < S;
  // this thread's threshold vector
  int32_t t[KM1];
  {
    const int64_t R = (int64_t)(1 << q) + 2;
    int64_t rem = valid ? s : 0;
#pragma unroll
    for (int k = KM1 - 1; k >= 0; --k) {
      if (bvecs) {
        t[k] = valid ? __ldg(bvecs + s * KM1 + k) : 0;
      } else {
        t[k] = (int32_t)(rem % R);
        rem /= R;
      }
    }
  }
  unsigned long long e = 0ull;
  uint32_t c = 0;
  uint32_t reach[K];
#pragma unroll
  for (int k = 0; k < K; ++k) reach[k] = 0;
  for (int64_t r0 = 0; r0 < N; r0 += kReplayTile) {
    const int m = (int)min((int64_t)kReplayTile, Np - r0);   // multiple of 4
    __syncthreads();
    for (int i = threadIdx.x * 4; i < m; i += kReplayThreads * 4) {
#pragma unroll
      for (int k = 0; k < KM1; ++k)
        *reinterpret_cast<int4*>(&sb[k][i]) = __ldg(reinterpret_cast<const int4*>(bins + (int64_t)k * Np + r0 + i));
      *reinterpret_cast<uint4*>(&sk[i]) = __ldg(reinterpret_cast<const uint4*>(bits + r0 + i));
    }
    __syncthreads();
    const int mr = (int)min((int64_t)m, N - r0);             // real samples in the tile
    int i = 0;
    for (; i + 4 <= mr; i += 4) {
      int4 b4[KM1];
#pragma unroll
      for (int k = 0; k < KM1; ++k) b4[k] = *reinterpret_cast<const int4*>(&sb[k][i]);
      const uint4 k4 = *reinterpret_cast<const uint4*>(&sk[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int st = KM1;                                        // the last model answers the rest
#pragma unroll
        for (int k = KM1 - 1; k >= 0; --k) {
          const int32_t bk = j == 0 ? b4[k].x : j == 1 ? b4[k].y : j == 2 ? b4[k].z : b4[k].w;
          if (bk >= t[k]) st = k;
        }
        const uint32_t kb = j == 0 ? k4.x : j == 1 ? k4.y : j == 2 ? k4.z : k4.w;
        c += (kb >> st) & 1u;
        e += scw[st];
        if (REACH) {
#pragma unroll
          for (int k = 1; k < K; ++k) reach[k] += st >= k ? 1u : 0u;
        }
      }
    }
    for (; i < mr; ++i) {
      int st = KM1;
#pragma unroll
      for (int k = KM1 - 1; k >= 0; --k)
        if (sb[k][i] >= t[k]) st = k;
      c += (sk[i] >> st) & 1u;
      e += scw[st];
      if (REACH) {
#pragma unroll
        for (int k = 1; k < K; ++k) reach[k] += st >= k ? 1u : 0u;
      }
    }
  }
  if (valid) {
    out_c[s] = (int64_t)c;
    out_e[s] = (int64_t)e;
    if (REACH) {
      out_reach[s * K] = N;
#pragma unroll
      for (int k = 1; k < K; ++k) out_reach[s * K + k] = (int64_t)reach[k];
    }
  }
}

// ---- K9b': prefix histograms for the exhaustive grid -------------------------
constexpr int kHistThreads = 256;
constexpr int kHistMaxR = 48;                  // B + 2 <= 48: q <= 5
constexpr int kPackBits = 21;                  // N < 2^21 per (prefix, bin) counter field

// hist[p][v] (v = bin_{K-2} + 1 in 0..R-1) packed count | correct_{K-2} << 21 |
// correct_{K-1} << 42; pre[p] = {correct, energy} of the requests answered by
// models 0..K-3; preach[p][k-1] = requests reaching model k (1 <= k <= K-2)
template <int KM1>
__global__ void __launch_bounds__(kHistThreads) replay_hist_kernel(
    const int32_t* __restrict__ bins, const uint32_t* __restrict__ bits, int64_t N, int64_t Np, int q,
    int64_t P, int64_t chunk, const __grid_constant__ ReplayWeights cw,
    unsigned long long* hist, unsigned long long* pre, unsigned long long* preach) {
  pdl_start();
  constexpr int KP = KM1 - 1;                               // compares before the last threshold
  constexpr int kTile = hist_tile(KM1);
  extern __shared__ __align__(16) unsigned char smraw[];
  int32_t* sb = reinterpret_cast<int32_t*>(smraw);           // [KM1][kTile]
  uint32_t* sk = reinterpret_cast<uint32_t*>(sb + (size_t)KM1 * kTile);
  unsigned long long* sh = reinterpret_cast<unsigned long long*>(sk + kTile);   // [R][kHistThreads]
  const int R = (1 << q) + 2;
  const int tid = threadIdx.x;
  const int64_t p = (int64_t)blockIdx.x * kHistThreads + tid;
  const bool valid = p < P;
  int32_t t[KP > 0 ? KP : 1];
  {
    int64_t rem = valid ? p : 0;
#pragma unroll
    for (int k = KP - 1; k >= 0; --k) {
      t[k] = (int32_t)(rem % R);
      rem /= R;
    }
  }
  for (int v = 0; v < R; ++v) sh[(size_t)v * kHistThreads + tid] = 0ull;
  unsigned long long a = 0ull;
  uint32_t reach[KP > 0 ? KP : 1];
#pragma unroll
  for (int k = 0; k < (KP > 0 ? KP : 1); ++k) reach[k] = 0;
  const int64_t s0 = (int64_t)blockIdx.y * chunk, s1 = min(N, s0 + chunk);
  for (int64_t r0 = s0; r0 < s1; r0 += kTile) {
    const int m = (int)min((int64_t)kTile, (s1 - r0 + 3) & ~(int64_t)3);
    __syncthreads();
    for (int i = tid * 4; i < m; i += kHistThreads * 4) {
#pragma unroll
      for (int k = 0; k < KM1; ++k)
        *reinterpret_cast<int4*>(&sb[(size_t)k * kTile + i]) =
            __ldg(reinterpret_cast<const int4*>(bins + (int64_t)k * Np + r0 + i));
      *reinterpret_cast<uint4*>(&sk[i]) = __ldg(reinterpret_cast<const uint4*>(bits + r0 + i));
    }
    __syncthreads();
    const int mr = (int)min((int64_t)m, s1 - r0);
    // one request: answering model among 0..K-3 (st < KP) or alive at K-2 (st == KP);
    // a counts correct_st for every request (the alive ones' correct_{K-2} total is
    // the histogram's, subtracted in the finish kernel), reach[k] = #(st > k)
    auto visit = [&](const int32_t (&bk)[KM1], uint32_t kb) {
      int st = KP;
#pragma unroll
      for (int k = KP - 1; k >= 0; --k)
        if (bk[k] >= t[k]) st = k;
      a += (kb >> st) & 1u;
#pragma unroll
      for (int k = 0; k < KP; ++k) reach[k] += st > k ? 1u : 0u;
      if (st == KP) {
        unsigned long long* h = sh + (size_t)(bk[KP] + 1) * kHistThreads + tid;   // bin + 1: 0 = NaN
        *h += 1ull | ((unsigned long long)((kb >> KP) & 1u) << kPackBits) |
              ((unsigned long long)((kb >> KM1) & 1u) << (2 * kPackBits));
      }
    };
    int i = 0;
    for (; i + 4 <= mr; i += 4) {
      int4 b4[KM1];
#pragma unroll
      for (int k = 0; k < KM1; ++k) b4[k] = *reinterpret_cast<const int4*>(&sb[(size_t)k * kTile + i]);
      const uint4 k4 = *reinterpret_cast<const uint4*>(&sk[i]);
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        int32_t bk[KM1];
#pragma unroll
        for (int k = 0; k < KM1; ++k) bk[k] = j == 0 ? b4[k].x : j == 1 ? b4[k].y : j == 2 ? b4[k].z : b4[k].w;
        visit(bk, j == 0 ? k4.x : j == 1 ? k4.y : j == 2 ? k4.z : k4.w);
      }
    }
    for (; i < mr; ++i) {
      int32_t bk[KM1];
#pragma unroll
      for (int k = 0; k < KM1; ++k) bk[k] = sb[(size_t)k * kTile + i];
      visit(bk, sk[i]);
    }
  }
  if (!valid) return;
  for (int v = 0; v < R; ++v) {
    const unsigned long long h = sh[(size_t)v * kHistThreads + tid];
    if (h) atomicAdd(hist + p * R + v, h);
  }
  if (a) atomicAdd(pre + 2 * p, a);
#pragma unroll
  for (int k = 0; k < KP; ++k)
    if (reach[k]) atomicAdd(preach + p * (KP > 0 ? KP : 1) + k, (unsigned long long)reach[k]);
}

// one thread per prefix: the R vectors (prefix, b) from prefix sums over its histogram
template <int KM1>
__global__ void __launch_bounds__(256) replay_finish_kernel(
    const unsigned long long* __restrict__ hist, const unsigned long long* __restrict__ pre,
    const unsigned long long* __restrict__ preach, int64_t N, int q, int64_t P,
    const __grid_constant__ ReplayWeights cw, int64_t* out_c, int64_t* out_e, int64_t* out_reach) {
  pdl_start();
  constexpr int KP = KM1 - 1;
  constexpr int K = KM1 + 1;
  const int R = (1 << q) + 2;
  const int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (p >= P) return;
  const unsigned long long mask = (1ull << kPackBits) - 1ull;
  unsigned long long tn = 0, ta = 0, tz = 0;
  for (int v = 0; v < R; ++v) {
    const unsigned long long h = hist[p * R + v];
    tn += h & mask;
    ta += (h >> kPackBits) & mask;
    tz += h >> (2 * kPackBits);
  }
  // requests answered by models 0..K-3: correct = a_all - (correct_{K-2} of the alive ones);
  // energy = sum_{k<K-2} w_k * (reach_k - alive), reach_0 = N
  const unsigned long long A = pre[2 * p] - ta;
  unsigned long long E = 0ull;
#pragma unroll
  for (int k = 0; k < KP; ++k) {
    const unsigned long long rk = k == 0 ? (unsigned long long)N : preach[p * (KP > 0 ? KP : 1) + k - 1];
    E += (cw.cum[k] - (k ? cw.cum[k - 1] : 0ull)) * (rk - tn);
  }
  const unsigned long long wa = cw.cum[KP], wz = cw.cum[KM1];
  unsigned long long dn = 0, da = 0, dz = 0;               // bins < b: deferred to the last model
  for (int b = 0; b < R; ++b) {
    const unsigned long long h = hist[p * R + b];           // v = b  <=>  bin = b - 1 < b
    dn += h & mask;
    da += (h >> kPackBits) & mask;
    dz += h >> (2 * kPackBits);
    const int64_t s = p * R + b;
    out_c[s] = (int64_t)(A + (ta - da) + dz);
    out_e[s] = (int64_t)(E + (tn - dn) * wa + dn * wz);
    if (out_reach) {
      out_reach[s * K] = N;
#pragma unroll
      for (int k = 0; k < KP; ++k) out_reach[s * K + 1 + k] = (int64_t)preach[p * (KP > 0 ? KP : 1) + k];
      out_reach[s * K + KM1] = (int64_t)dn;
    }
  }
}

__global__ void zero_u64_kernel(unsigned long long* p, int64_t n) {
  pdl_start();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = 0ull;
}

template <int KM1>
cudaError_t launch_replay_hist_k(const ReplayArgs& a, unsigned long long* hws, cudaStream_t s) {
  constexpr int KP = KM1 - 1;
  const int R = (1 << a.q) + 2;
  const int64_t P = a.S / R;
  unsigned long long* hist = hws;
  unsigned long long* pre = hist + (size_t)P * R;
  unsigned long long* preach = pre + 2 * (size_t)P;
  const int64_t nz = (int64_t)P * R + 2 * P + P * (KP > 0 ? KP : 1);
  cudaError_t e = launch_pdl(zero_u64_kernel, dim3((unsigned)min((int64_t)num_sms() * 4, (nz + 255) / 256)),
                             dim3(256), 0, s, hws, nz);
  if (e != cudaSuccess) return e;
  auto kern = replay_hist_kernel<KM1>;
  const size_t smem = ((size_t)KM1 * hist_tile(KM1) + hist_tile(KM1)) * 4 +
                      (size_t)R * kHistThreads * 8;
  static bool attr[8] = {};
  if (!attr[KM1]) {
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    attr[KM1] = true;
  }
  const int64_t pb = (P + kHistThreads - 1) / kHistThreads;
  int per_sm = 1;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kHistThreads, smem);
  // split the samples so that the grid fills the GPU about twice (>= 1024 samples per CTA)
  int64_t chunks = max((int64_t)1, (int64_t)num_sms() * max(per_sm, 1) * 2 / pb);
  chunks = min(chunks, max((int64_t)1, a.N / 1024));
  int64_t chunk = (a.N + chunks - 1) / chunks;
  chunk = (chunk + 3) / 4 * 4;
  chunks = (a.N + chunk - 1) / chunk;
  e = launch_pdl(kern, dim3((unsigned)pb, (unsigned)chunks), dim3(kHistThreads), smem, s, a.bins, a.bits,
                 a.N, a.Np, a.q, P, chunk, a.w, hist, pre, preach);
  if (e != cudaSuccess) return e;
  return launch_pdl(replay_finish_kernel<KM1>, dim3((unsigned)((P + 255) / 256)), dim3(256), 0, s,
                    (const unsigned long long*)hist, (const unsigned long long*)pre,
                    (const unsigned long long*)preach, a.N, a.q, P, a.w, a.out_c, a.out_e, a.reach);
}

// ---- K9c: frontier -------------------------------------------------------------
__global__ void graph_init_kernel(unsigned long long* minE, long long* minS, int64_t n1) {
  pdl_start();
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n1; i += (int64_t)gridDim.x * blockDim.x) {
    minE[i] = ~0ull;
    minS[i] = LLONG_MAX;
  }
}

__global__ void graph_min_kernel(const int64_t* __restrict__ C, const int64_t* __restrict__ E, int64_t S,
                                 int64_t n1, unsigned long long* minE, uint32_t* status) {
  pdl_start();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = C[s];
    if (c < 0 || c >= n1 || E[s] < 0) {
      if (status) atomicOr(status, HS_STATUS_NONFINITE);
      continue;
    }
    atomicMin(minE + c, (unsigned long long)E[s]);
  }
}

__global__ void graph_rep_kernel(const int64_t* __restrict__ C, const int64_t* __restrict__ E, int64_t S,
                                 int64_t n1, const unsigned long long* minE, long long* minS) {
  pdl_start();
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < S; s += (int64_t)gridDim.x * blockDim.x) {
    const int64_t c = C[s];
    if (c < 0 || c >= n1 || E[s] < 0) continue;
    if ((unsigned long long)E[s] == minE[c]) atomicMin(minS + c, (long long)s);
  }
}

template <typename T, typename Op>
__device__ T block_scan_incl(T v, T* sh, Op op) {   // inclusive scan over threadIdx order
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const T u = __shfl_up_sync(0xFFFFFFFFu, v, o);
    if (lane >= o) v = op(u, v);
  }
  if (lane == 31) sh[warp] = v;
  __syncthreads();
  if (warp == 0) {
    T w = sh[lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const T u = __shfl_up_sync(0xFFFFFFFFu, w, o);
      if (lane >= o) w = op(u, w);
    }
    sh[lane] = w;
  }
  __syncthreads();
  if (warp > 0) v = op(sh[warp - 1], v);
  __syncthreads();
  return v;
}

struct AddOp {
  __device__ long long operator()(long long a, long long b) const { return a + b; }
};

// One CTA.  Thread t owns counts [t*chunk, (t+1)*chunk).  Kept(c) <=> minE[c] <
// min_{c' > c} minE[c'] (strict: a count with no vector has minE = ~0).
__global__ void __launch_bounds__(kFrontThreads) graph_front_kernel(
    const unsigned long long* __restrict__ minE, const long long* __restrict__ minS, int64_t n1,
    int64_t tau, int64_t floor_, const unsigned long long* model_correct, int K,
    int64_t* front_c, int64_t* front_e, int64_t* front_s, int64_t* front_n, int64_t* pick) {
  pdl_start();
  __shared__ long long shl[32];
  __shared__ double shd[32];
  __shared__ long long shj[32];
  __shared__ long long s_ap, s_n;
  const int tid = threadIdx.x;
  const int T = kFrontThreads;
  if (tau < 0) tau = model_correct ? (int64_t)model_correct[K - 1] : 0;
  if (floor_ < 0) floor_ = model_correct ? (int64_t)model_correct[K - 2] : 0;
  // Tiles of kFrontTile counts from the top down (coalesced loads into shared
  // memory; thread t owns kFrontTE consecutive counts of the tile).  Kept(c) <=>
  // minE[c] < min over every larger count; kept points are written in
  // DESCENDING c first (their positions are known from the top), then reversed.
  __shared__ unsigned long long tv[kFrontTile];
  __shared__ unsigned long long cmin[kFrontThreads];
  unsigned long long carry = ~0ull;                         // min over the tiles above
  long long J = 0;
  for (int64_t t0 = ((n1 - 1) / kFrontTile) * kFrontTile; n1 > 0 && t0 >= 0; t0 -= kFrontTile) {
    for (int i = tid; i < kFrontTile; i += T) tv[i] = (t0 + i < n1) ? minE[t0 + i] : ~0ull;
    __syncthreads();
    unsigned long long cm = ~0ull;
#pragma unroll
    for (int j = 0; j < kFrontTE; ++j) cm = min(cm, tv[tid * kFrontTE + j]);
    cmin[tid] = cm;
    __syncthreads();
    for (int o = 1; o < T; o <<= 1) {                       // suffix minimum over the threads
      const unsigned long long v = (tid + o < T) ? cmin[tid + o] : ~0ull;
      __syncthreads();
      cmin[tid] = min(cmin[tid], v);
      __syncthreads();
    }
    const unsigned long long above = min(carry, (tid + 1 < T) ? cmin[tid + 1] : ~0ull);
    unsigned kmask = 0;
    long long kept = 0;
    {
      unsigned long long run = above;
#pragma unroll
      for (int j = kFrontTE - 1; j >= 0; --j) {
        const unsigned long long v = tv[tid * kFrontTE + j];
        if (v < run) {
          kmask |= 1u << j;
          ++kept;
          run = v;
        }
      }
    }
    const long long incl = block_scan_incl<long long>(kept, shl, AddOp());
    if (tid == T - 1) s_n = incl;                           // kept in this tile
    __syncthreads();
    const long long tile_kept = s_n;
    long long pos = J + (tile_kept - incl);                 // kept points of higher threads come first
#pragma unroll
    for (int j = kFrontTE - 1; j >= 0; --j) {
      if (kmask & (1u << j)) {
        const int64_t c = t0 + tid * kFrontTE + j;
        front_c[pos] = c;
        front_e[pos] = (int64_t)tv[tid * kFrontTE + j];
        front_s[pos] = (int64_t)minS[c];
        ++pos;
      }
    }
    J += tile_kept;
    carry = min(carry, cmin[0]);
    __syncthreads();
  }
  // ascending c: reverse the J points in place (disjoint pairs)
  for (long long i = tid; i < J / 2; i += T) {
    const long long k = J - 1 - i;
    const int64_t c0 = front_c[i], e0 = front_e[i], s0 = front_s[i];
    front_c[i] = front_c[k];
    front_e[i] = front_e[k];
    front_s[i] = front_s[k];
    front_c[k] = c0;
    front_e[k] = e0;
    front_s[k] = s0;
  }
  if (tid == 0) {
    s_ap = -1;
    s_n = J;
  }
  __syncthreads();
  // 4. AP: the first frontier point with c >= tau
  for (long long j = tid; j < J; j += T) {
    if (front_c[j] >= tau && (j == 0 || front_c[j - 1] < tau)) s_ap = front_s[j];
  }
  // 5. EO: largest second divided difference among interior points with c >= floor
  double bd = -INFINITY;
  long long bj = LLONG_MAX;
  for (long long j = 1 + tid; j + 1 < J; j += T) {
    if (front_c[j] < floor_) continue;
    const double d1 = __ddiv_rn((double)(front_e[j + 1] - front_e[j]), (double)(front_c[j + 1] - front_c[j]));
    const double d0 = __ddiv_rn((double)(front_e[j] - front_e[j - 1]), (double)(front_c[j] - front_c[j - 1]));
    const double d = __dsub_rn(d1, d0);
    if (d > bd) {                                          // ascending j: ties keep the lowest
      bd = d;
      bj = j;
    }
  }
  const int lane = tid & 31, warp = tid >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const double od = __shfl_xor_sync(0xFFFFFFFFu, bd, o);
    const long long oj = __shfl_xor_sync(0xFFFFFFFFu, bj, o);
    if (od > bd || (od == bd && oj < bj)) {
      bd = od;
      bj = oj;
    }
  }
  if (lane == 0) {
    shd[warp] = bd;
    shj[warp] = bj;
  }
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < T / 32; ++w)
      if (shd[w] > bd || (shd[w] == bd && shj[w] < bj)) {
        bd = shd[w];
        bj = shj[w];
      }
    *front_n = J;
    pick[0] = s_ap;
    pick[1] = bj != LLONG_MAX ? front_s[bj] : s_ap;       // no interior candidate: EO = AP
  }
}

template <int KM1>
cudaError_t launch_replay_k(const ReplayArgs& a, cudaStream_t s) {
  const int64_t blocks = (a.S + kReplayThreads - 1) / kReplayThreads;
  if (a.reach)
    return launch_pdl(replay_kernel<KM1, true>, dim3((unsigned)blocks), dim3(kReplayThreads), 0, s,
                      a.bins, a.bits, a.N, a.Np, a.q, a.bvecs, a.S, a.w, a.out_c, a.out_e, a.reach);
  return launch_pdl(replay_kernel<KM1, false>, dim3((unsigned)blocks), dim3(kReplayThreads), 0, s,
                    a.bins, a.bits, a.N, a.Np, a.q, a.bvecs, a.S, a.w, a.out_c, a.out_e, a.reach);
}

}  // namespace

// the exhaustive grid goes through the prefix histograms when they fit
static bool use_hist(int K, int q, int64_t N) {
  static const bool direct = getenv("HS_REPLAY_DIRECT") && getenv("HS_REPLAY_DIRECT")[0] == '1';
  return !direct && (1 << q) + 2 <= kHistMaxR && N < (int64_t(1) << kPackBits) && K >= 2;
}
static size_t hist_ws_bytes(int K, int q) {
  const int64_t R = (1 << q) + 2;
  int64_t P = 1;
  for (int k = 0; k < K - 2; ++k) P *= R;
  return (size_t)(P * R + 2 * P + P * (K > 2 ? K - 2 : 1)) * 8u;
}

size_t replay_ws_bytes(int K, int64_t N, int q) {
  const int64_t Np = (N + 3) / 4 * 4;
  size_t b = ((size_t)Np * (size_t)K * 4u + 255u) / 256u * 256u + 256u;
  if (use_hist(K, q, N)) b += hist_ws_bytes(K, q);
  return b;
}

cudaError_t launch_replay(ReplayArgs a, const float* conf, const uint8_t* correct,
                          unsigned long long* model_correct, void* ws, cudaStream_t s) {
  a.Np = (a.N + 3) / 4 * 4;
  a.bins = reinterpret_cast<int32_t*>(ws);
  a.bits = reinterpret_cast<uint32_t*>(a.bins + (size_t)(a.K - 1) * a.Np);
  cudaError_t e;
  if (model_correct) {
    e = launch_pdl(replay_zero_kernel, dim3(1), dim3(32), 0, s, model_correct, a.K);
    if (e != cudaSuccess) return e;
  }
  int blocks = (int)min((int64_t)num_sms() * 4, (a.Np + 255) / 256);
  if (blocks < 1) blocks = 1;
  e = launch_pdl(replay_prep_kernel, dim3(blocks), dim3(256), 0, s, conf, correct, a.K, a.N, a.Np,
                 a.q, a.bins, a.bits, model_correct);
  if (e != cudaSuccess || a.S == 0) return e;
  if (!a.bvecs && use_hist(a.K, a.q, a.N)) {
    unsigned long long* hws = reinterpret_cast<unsigned long long*>(
        reinterpret_cast<char*>(ws) + ((size_t)a.Np * (size_t)a.K * 4u + 255u) / 256u * 256u + 256u);
    switch (a.K - 1) {
      case 1: return launch_replay_hist_k<1>(a, hws, s);
      case 2: return launch_replay_hist_k<2>(a, hws, s);
      case 3: return launch_replay_hist_k<3>(a, hws, s);
      case 4: return launch_replay_hist_k<4>(a, hws, s);
      case 5: return launch_replay_hist_k<5>(a, hws, s);
      case 6: return launch_replay_hist_k<6>(a, hws, s);
      case 7: return launch_replay_hist_k<7>(a, hws, s);
      default: return cudaErrorInvalidValue;
    }
  }
  switch (a.K - 1) {
    case 1: return launch_replay_k<1>(a, s);
    case 2: return launch_replay_k<2>(a, s);
    case 3: return launch_replay_k<3>(a, s);
    case 4: return launch_replay_k<4>(a, s);
    case 5: return launch_replay_k<5>(a, s);
    case 6: return launch_replay_k<6>(a, s);
    case 7: return launch_replay_k<7>(a, s);
    default: return cudaErrorInvalidValue;
  }
}

size_t graph_ws_bytes(int64_t N) { return (size_t)(N + 1) * 16u + 256u; }

cudaError_t launch_graph(const int64_t* C, const int64_t* E, int64_t S, int64_t N, int64_t tau,
                         int64_t floor_, const unsigned long long* model_correct, int K,
                         int64_t* front_c, int64_t* front_e, int64_t* front_s, int64_t* front_n,
                         int64_t* pick, uint32_t* status, void* ws, cudaStream_t s) {
  const int64_t n1 = N + 1;
  unsigned long long* minE = reinterpret_cast<unsigned long long*>(ws);
  long long* minS = reinterpret_cast<long long*>(minE + n1);
  const int gi = (int)min((int64_t)num_sms() * 4, (n1 + 255) / 256);
  const int gs = (int)max((int64_t)1, min((int64_t)num_sms() * 8, (S + 255) / 256));
  cudaError_t e = launch_pdl(graph_init_kernel, dim3(gi), dim3(256), 0, s, minE, minS, n1);
  if (e != cudaSuccess) return e;
  e = launch_pdl(graph_min_kernel, dim3(gs), dim3(256), 0, s, C, E, S, n1, minE, status);
  if (e != cudaSuccess) return e;
  e = launch_pdl(graph_rep_kernel, dim3(gs), dim3(256), 0, s, C, E, S, n1,
                 (const unsigned long long*)minE, minS);
  if (e != cudaSuccess) return e;
  return launch_pdl(graph_front_kernel, dim3(1), dim3(kFrontThreads), 0, s,
                    (const unsigned long long*)minE, (const long long*)minS, n1, tau, floor_,
                    model_correct, K, front_c, front_e, front_s, front_n, pick);
}

}  // namespace hs
