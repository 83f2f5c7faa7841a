// conf.cu -- K1 (per-row confidence) and K2 (token -> sequence reduce).
//
// The confidence score function of HybridServe applied to the
// logits of one stage model: temperature-scaled softmax (TS) in one
// pass over HBM, giving per row
//     m = max_j x_j,  a_j = (x_j - m) * log2(e) / T,  s = sum_j 2^{a_j},
//     w = sum_j 2^{a_j} a_j,  p_max = 1/s,  H = ln s - ln2 * w / s,
//     argmax = lowest j with x_j = m,
// and the confidence c = p_max | p_max^2 | exp(-H) (readings G1/G3).
//
// Bandwidth-bound: each logit is read once with 128-bit streaming loads; the
// per-element work is ~4 issue slots (bf16 unpack, FADD2/FMUL2 on packed fp32
// pairs, one MUFU.EX2 per element, FADD2/FFMA2 accumulation).  (x - m) is
// formed exactly before scaling so the 1e-5 relative confidence tolerance holds
// even at T = 0.05.
//
// Two launch shapes:
//   * conf_warp_kernel  -- one warp per row, the whole row in registers
//     (C <= 4096 bf16 / 2048 fp32: ViT/GLUE classifiers).  Exact two-step
//     (row max by shuffle, then exponentials) -- no online rescaling.  The next
//     row's loads are issued before the current row is reduced.
//   * conf_cta_kernel   -- one CTA per row, persistent over rows, per-thread
//     online (max, sum, weighted sum) over 8-vector chunks, block merge
//     (vocabulary-sized rows: T5 32,128, Llama 128,256).
#include <cuda_bf16.h>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace {

struct RowOut {
  float m;     // raw row max (NaN / +inf / -inf => invalid row)
  float s;     // sum 2^a
  float w;     // sum 2^a * a
  uint32_t am; // argmax
};

__device__ __forceinline__ void write_row(const ConfArgs& a, int64_t row, int64_t src_row,
                                          const RowOut& r) {
  const bool bad = !(r.m < INFINITY) || (r.m == -INFINITY);
  float c;
  int32_t am = (int32_t)r.am;
  if (bad) {
    c = __int_as_float(0x7FC00000);
    am = -1;
    if (a.status) atomicOr(a.status, HS_STATUS_NONFINITE);
  } else {
    const float p = 1.0f / r.s;
    if (a.kind == HS_CONF_MAXPROB_SQ) {
      c = p * p;
    } else if (a.kind == HS_CONF_ENTROPY) {
      // exp(-H) = (1/s) * 2^{w/s} = 2^{w/s - log2 s}; full-precision exp2f/log2f
      c = exp2f(r.w / r.s - log2f(r.s));
    } else {
      c = p;
    }
  }
  a.conf[row] = c;
  if (a.argmax) a.argmax[row] = am;
  if (a.ok) a.ok[row] = (uint8_t)(a.labels ? (!bad && a.labels[src_row] == am) : 0);
}

__device__ __forceinline__ int64_t source_row(const ConfArgs& a, int64_t row) {
  if (!a.row_index) return row;
  if (a.L == 1) return a.row_index[row];
  return a.row_index[row / a.L] * a.L + row % a.L;
}

__device__ __forceinline__ int64_t live_rows(const ConfArgs& a) {
  int64_t n = a.n;
  if (a.d_n) {
    int64_t dn = *a.d_n;
    n = dn < n ? dn : n;
  }
  return n * a.L;
}

// -inf for out-of-row lanes of the last partial 16-byte vector
template <bool BF16>
__device__ __forceinline__ void mask_tail(uint4& v, int tail) {
  uint32_t* w = reinterpret_cast<uint32_t*>(&v);
  if (BF16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      if (2 * q >= tail) w[q] = kBf16NegInf2;
      else if (2 * q + 1 >= tail) w[q] = (w[q] & 0xFFFFu) | 0xFF800000u;
    }
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q)
      if (q >= tail) w[q] = kF32NegInf;
  }
}

template <bool BF16>
__device__ __forceinline__ uint4 load_vec(const uint4* p, int vi, int nvec, int tail) {
  uint4 v;
  if (vi < nvec) {
    v = ldg_stream(p + vi);
    if (tail && vi == nvec - 1) mask_tail<BF16>(v, tail);
  } else {
    const uint32_t f = BF16 ? kBf16NegInf2 : kF32NegInf;
    v = make_uint4(f, f, f, f);
  }
  return v;
}

// NaN-propagating max of one 16-byte vector (as fp32)
template <bool BF16>
__device__ __forceinline__ float vec_max(const uint4& v) {
  if (BF16) {
    uint32_t t = bmax2(bmax2(v.x, v.y), bmax2(v.z, v.w));
    return fmax_nan(bf_lo(t), bf_hi(t));
  } else {
    return fmax3_nan(__uint_as_float(v.x), __uint_as_float(v.y),
                     fmax_nan(__uint_as_float(v.z), __uint_as_float(v.w)));
  }
}

// first element (0..VE-1) of v equal to m, VE if none
template <bool BF16>
__device__ __forceinline__ int vec_first_eq(const uint4& v, float m) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
  int r = BF16 ? 8 : 4;
  if (BF16) {
#pragma unroll
    for (int q = 3; q >= 0; --q) {
      if (bf_hi(w[q]) == m) r = 2 * q + 1;
      if (bf_lo(w[q]) == m) r = 2 * q;
    }
  } else {
#pragma unroll
    for (int q = 3; q >= 0; --q)
      if (__uint_as_float(w[q]) == m) r = q;
  }
  return r;
}

// Accumulate 2^a and 2^a * a of one vector into the packed accumulators.
template <bool BF16, bool ENTROPY>
__device__ __forceinline__ void vec_accum(const uint4& v, f2_t m2, f2_t c2, uint32_t clampw,
                                          f2_t& s2, f2_t& w2) {
  const uint32_t* w = reinterpret_cast<const uint32_t*>(&v);
  if (BF16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t u = ENTROPY ? bmax2_plain(w[q], clampw) : w[q];
      f2_t a = f2mul(f2sub(f2(bf_lo(u), bf_hi(u)), m2), c2);
      f2_t e = f2(ex2(f2lo(a)), ex2(f2hi(a)));
      s2 = f2add(s2, e);
      if (ENTROPY) w2 = f2fma(e, a, w2);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      f2_t a = f2mul(f2sub(f2(__uint_as_float(w[2 * q]), __uint_as_float(w[2 * q + 1])), m2), c2);
      float a0 = f2lo(a), a1 = f2hi(a);
      if (ENTROPY) {  // -inf (masked) logits: keep 2^a * a = 0 instead of 0 * -inf
        a0 = fmaxf(a0, -128.f);
        a1 = fmaxf(a1, -128.f);
        a = f2(a0, a1);
      }
      f2_t e = f2(ex2(a0), ex2(a1));
      s2 = f2add(s2, e);
      if (ENTROPY) w2 = f2fma(e, a, w2);
    }
  }
}

// bf16x2 word holding a lower bound L <= m - 128/c (rounded down): clamping
// x >= L leaves every term with 2^a >= 2^-128 untouched and turns -inf into a
// finite value whose 2^a flushes to 0, so 2^a * a stays 0 (masked classes).
// The offset is at least |m| * 2^-7 so that m - offset is never absorbed by
// fp32 rounding (which would clamp everything to m).
__device__ __forceinline__ uint32_t entropy_clamp_word(float m, float c) {
  const float off = fmaxf(128.0f / c, fabsf(m) * 0.0078125f);
  __nv_bfloat16 b = __float2bfloat16_rd(m - off);
  uint32_t u = (uint32_t)__bfloat16_as_ushort(b);
  return u | (u << 16);
}

// ---------------------------------------------------------------------------
// K1a: one warp per row, row in registers.
// ---------------------------------------------------------------------------
template <bool BF16, bool ENTROPY, int NV>
__global__ void __launch_bounds__(256) conf_warp_kernel(const ConfArgs a) {
  const int lane = threadIdx.x & 31;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int64_t rows = live_rows(a);
  const float c = a.c;
  const f2_t c2 = f2(c, c);
  constexpr int VE = BF16 ? 8 : 4;

  int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (row >= rows) return;
  int64_t src = source_row(a, row);
  uint4 v[NV];
  {
    const uint4* p = reinterpret_cast<const uint4*>((const char*)a.logits + src * a.row_bytes);
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = load_vec<BF16>(p, k * 32 + lane, a.nvec, a.tail);
  }
  while (true) {
    // prefetch the next row before reducing this one
    const int64_t nrow = row + nwarps;
    const bool more = nrow < rows;
    int64_t nsrc = 0;
    uint4 nv[NV];
    if (more) {
      nsrc = source_row(a, nrow);
      const uint4* p = reinterpret_cast<const uint4*>((const char*)a.logits + nsrc * a.row_bytes);
#pragma unroll
      for (int k = 0; k < NV; ++k) nv[k] = load_vec<BF16>(p, k * 32 + lane, a.nvec, a.tail);
    }

    // 1. row max (exact, NaN-propagating)
    float vm[NV];
    float lm = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      vm[k] = vec_max<BF16>(v[k]);
      lm = fmax_nan(lm, vm[k]);
    }
    float m = lm;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));

    // 2. argmax: first vector holding m (lowest vector index), then first element in it
    unsigned my_vi = 0xFFFFFFFFu;
#pragma unroll
    for (int k = NV - 1; k >= 0; --k)
      if (vm[k] == m) my_vi = (unsigned)(k * 32 + lane);
    const unsigned vstar = __reduce_min_sync(0xFFFFFFFFu, my_vi);
    unsigned am = 0;
    if (vstar != 0xFFFFFFFFu) {
      const int owner = (int)(vstar & 31u), kstar = (int)(vstar >> 5);
      int e = 0;
      if (lane == owner) {
        uint4 sel = v[0];
#pragma unroll
        for (int k = 1; k < NV; ++k)
          if (k == kstar) sel = v[k];
        e = vec_first_eq<BF16>(sel, m);
      }
      e = __shfl_sync(0xFFFFFFFFu, e, owner);
      am = vstar * VE + (unsigned)e;
    }

    // 3. exponentials with the common max
    f2_t s2 = f2(0.f, 0.f), w2 = f2(0.f, 0.f);
    const bool valid = (m < INFINITY) && (m > -INFINITY);
    if (valid) {
      const f2_t m2 = f2(m, m);
      const uint32_t cw = ENTROPY && BF16 ? entropy_clamp_word(m, c) : 0u;
#pragma unroll
      for (int k = 0; k < NV; ++k) vec_accum<BF16, ENTROPY>(v[k], m2, c2, cw, s2, w2);
    }
    float s = warp_sum(f2lo(s2) + f2hi(s2));
    float w = ENTROPY ? warp_sum(f2lo(w2) + f2hi(w2)) : 0.f;
    if (lane == 0) {
      RowOut r{m, s, w, am};
      write_row(a, row, src, r);
    }
    if (!more) break;
    row = nrow;
    src = nsrc;
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = nv[k];
  }
}

// ---------------------------------------------------------------------------
// K1b: one CTA per row (persistent over rows), per-thread online softmax.
// ---------------------------------------------------------------------------
template <bool BF16, bool ENTROPY, int NT, int NV>
__global__ void __launch_bounds__(NT) conf_cta_kernel(const ConfArgs a) {
  constexpr int NW = NT / 32;
  constexpr int VE = BF16 ? 8 : 4;
  __shared__ float sh_m[NW], sh_s[NW], sh_w[NW];
  __shared__ unsigned sh_am[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rows = live_rows(a);
  const float c = a.c;
  const f2_t c2 = f2(c, c);

  for (int64_t row = blockIdx.x; row < rows; row += gridDim.x) {
    const int64_t src = source_row(a, row);
    const uint4* p = reinterpret_cast<const uint4*>((const char*)a.logits + src * a.row_bytes);
    float m = -INFINITY;
    f2_t s2 = f2(0.f, 0.f), w2 = f2(0.f, 0.f);
    unsigned am = 0xFFFFFFFFu;
    for (int base = 0; base < a.nvec; base += NT * NV) {
      uint4 v[NV];
#pragma unroll
      for (int k = 0; k < NV; ++k) v[k] = load_vec<BF16>(p, base + k * NT + tid, a.nvec, a.tail);
      float cm = -INFINITY;
#pragma unroll
      for (int k = 0; k < NV; ++k) cm = fmax_nan(cm, vec_max<BF16>(v[k]));
      if (!(cm <= m)) {  // new running max (or NaN): rescale, locate its first index
        const float nm = fmax_nan(m, cm);
        if (m > -INFINITY) {
          const float d = (m - nm) * c;
          const float f = ex2(d);
          const f2_t f2v = f2(f, f);
          if (ENTROPY) w2 = f2mul(f2v, f2fma(f2(d, d), s2, w2));
          s2 = f2mul(f2v, s2);
        }
        m = nm;
        unsigned first = 0xFFFFFFFFu;
#pragma unroll
        for (int k = NV - 1; k >= 0; --k) {
          const int e = vec_first_eq<BF16>(v[k], cm);
          if (e < VE) first = (unsigned)((base + k * NT + tid) * VE + e);
        }
        am = first;
      }
      if (m > -INFINITY) {
        const f2_t m2 = f2(m, m);
        const uint32_t cw = ENTROPY && BF16 ? entropy_clamp_word(m, c) : 0u;
#pragma unroll
        for (int k = 0; k < NV; ++k) vec_accum<BF16, ENTROPY>(v[k], m2, c2, cw, s2, w2);
      }
    }
    // ---- block merge: max, rescale to it, fixed-order sums, min index among maxima
    float M = m;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) M = fmax_nan(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
    if (lane == 0) sh_m[wid] = M;
    __syncthreads();
    M = sh_m[0];
#pragma unroll
    for (int i = 1; i < NW; ++i) M = fmax_nan(M, sh_m[i]);
    float s = 0.f, w = 0.f;
    if (m > -INFINITY) {
      const float d = (m - M) * c;
      const float f = ex2(d);
      const float ls = f2lo(s2) + f2hi(s2);
      s = f * ls;
      if (ENTROPY && f > 0.f) w = f * ((f2lo(w2) + f2hi(w2)) + d * ls);
    }
    s = warp_sum(s);
    if (ENTROPY) w = warp_sum(w);
    const unsigned mine = (m == M) ? am : 0xFFFFFFFFu;
    const unsigned wam = __reduce_min_sync(0xFFFFFFFFu, mine);
    if (lane == 0) {
      sh_s[wid] = s;
      sh_w[wid] = w;
      sh_am[wid] = wam;
    }
    __syncthreads();
    if (tid == 0) {
      float S = 0.f, W = 0.f;
      unsigned A = 0xFFFFFFFFu;
#pragma unroll
      for (int i = 0; i < NW; ++i) {
        S += sh_s[i];
        W += sh_w[i];
        A = min(A, sh_am[i]);
      }
      RowOut r{M, S, W, A};
      write_row(a, row, src, r);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// K2: token -> sequence reduce, fixed order (P:423 MIN; MEAN), all-L correctness.
// ---------------------------------------------------------------------------
__global__ void seq_reduce_kernel(const float* tok_conf, const uint8_t* tok_ok, int64_t n,
                                  const int64_t* d_n, int L, int reduce, float* conf,
                                  uint8_t* correct) {
  int64_t live = n;
  if (d_n) live = min(*d_n, n);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < live;
       i += (int64_t)gridDim.x * blockDim.x) {
    const float* tc = tok_conf + i * L;
    float mn = INFINITY;
    double sum = 0.0;
    bool nan = false;
    uint8_t ok = 1;
    for (int t = 0; t < L; ++t) {
      const float x = tc[t];
      nan |= (x != x);
      mn = fminf(mn, x);
      sum += (double)x;
      if (tok_ok) ok &= tok_ok[i * L + t];
    }
    float r = (reduce == HS_SEQ_MEAN) ? (float)(sum / (double)L) : mn;
    if (nan) r = __int_as_float(0x7FC00000);
    conf[i] = r;
    if (correct) correct[i] = tok_ok ? ok : 0;
  }
}

template <typename K>
int occupancy(K kernel, int threads) {
  int b = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, kernel, threads, 0);
  return b > 0 ? b : 1;
}

template <bool BF16, bool ENTROPY, int NV>
cudaError_t launch_warp(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_warp_kernel<BF16, ENTROPY, NV>;
  static int occ = occupancy(k, 256);
  const int64_t want = (rows + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  k<<<grid, 256, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <bool BF16, bool ENTROPY, int NT>
cudaError_t launch_cta(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_cta_kernel<BF16, ENTROPY, NT, 8>;
  static int occ = occupancy(k, NT);
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(rows < cap ? (rows > 0 ? rows : 1) : cap);
  k<<<grid, NT, 0, s>>>(a);
  count_launch();
  return cudaGetLastError();
}

template <bool BF16, bool ENTROPY>
cudaError_t dispatch(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  const int nvec = a.nvec;
  if (nvec <= 32) return launch_warp<BF16, ENTROPY, 1>(a, rows, s);
  if (nvec <= 64) return launch_warp<BF16, ENTROPY, 2>(a, rows, s);
  if (nvec <= 128) return launch_warp<BF16, ENTROPY, 4>(a, rows, s);
  if (nvec <= 256) return launch_warp<BF16, ENTROPY, 8>(a, rows, s);
  if (nvec <= 512) return launch_warp<BF16, ENTROPY, 16>(a, rows, s);
  if (nvec <= 8192) return launch_cta<BF16, ENTROPY, 256>(a, rows, s);
  return launch_cta<BF16, ENTROPY, 512>(a, rows, s);
}

}  // namespace

const char* confidence_path(int64_t nvec) {
  if (nvec <= 512) return "warp-per-row";
  return "cta-per-row";
}

cudaError_t launch_confidence(const ConfArgs& a, bool bf16, cudaStream_t s) {
  const int64_t rows = a.n * a.L;
  const bool ent = a.kind == HS_CONF_ENTROPY;
  if (bf16) return ent ? dispatch<true, true>(a, rows, s) : dispatch<true, false>(a, rows, s);
  return ent ? dispatch<false, true>(a, rows, s) : dispatch<false, false>(a, rows, s);
}

cudaError_t launch_seq_reduce(const float* tok_conf, const uint8_t* tok_ok, int64_t n,
                              const int64_t* d_n, int L, int reduce, float* conf,
                              uint8_t* correct, cudaStream_t s) {
  const int64_t want = (n + 255) / 256;
  const int grid = (int)(want < 4096 ? (want > 0 ? want : 1) : 4096);
  seq_reduce_kernel<<<grid, 256, 0, s>>>(tok_conf, tok_ok, n, d_n, L, reduce, conf, correct);
  count_launch();
  return cudaGetLastError();
}

}  // namespace hs
