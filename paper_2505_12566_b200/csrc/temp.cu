// temp.cu -- NEXT-3: temperature fitting, Eq. 1.
//
// Temperature Scaling learns one T per stage model by minimising
// the NLL between the temperature-scaled softmax and the labels of the
// validation set:
//     NLL(T) = (1/n) sum_i [ LSE_j(x_ij / T) - x_{i,y_i} / T ].
// With beta = 1/T and d_ij = x_ij - m_i (m_i = row max), per row
//     nll_i = ln s_i - beta * dy_i,   s_i = sum_j e^{beta d_ij},   dy_i = x_{i,y_i} - m_i
//     g_i   = dnll_i/dbeta   = E_p[d_i] - dy_i
//     h_i   = d2nll_i/dbeta2 = Var_p[d_i] >= 0,
// so NLL is convex in beta and its minimiser over the clamp range
// [t_lo, t_hi] is where the mean of g changes sign, or a clamp end.
//
// Structure exploited here: m_i, dy_i and row validity do not depend on T, so
// they are computed once (sweep 0, 8 bytes per row to the workspace); every
// later sweep is ONE pass over the logits at one beta per stage model giving
// (sum nll, sum g, sum h) -- one MUFU ex2 and ~5 issue slots per logit.  A
// safeguarded Newton iteration on beta (Newton inside the bracket, probe of an
// unvisited clamp end, geometric bisection when a step does not halve) needs
// ~4-6 sweeps.  All sweeps of all stage models run in ONE persistent
// cooperative launch (one 1024-thread CTA per SM): per sweep every CTA writes
// its per-stage partial sums, one grid barrier, then EVERY CTA reduces the
// partials in the same fixed order and runs the identical update (no second
// barrier, no broadcast; deterministic bitwise).  Per-row sums are fp32
// (exact x - m, MUFU ex2), cross-row sums fp64.
#include <cooperative_groups.h>

#include <cmath>
#include <cstdlib>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace cg = cooperative_groups;

namespace {

#ifndef HS_TF_THREADS
#define HS_TF_THREADS 1024
#endif
constexpr int kTfThreads = HS_TF_THREADS;
constexpr int kTfWarps = kTfThreads / 32;
constexpr int kTfComp = 4;              // partial sums per stage: used, nll, g, h
// warm start: up to kTfSubPasses Newton sweeps over every kTfSubStride-th row
// (same objective on a 1/16 sample) before the first full sweep, for stages
// with >= kTfSubMin rows whose rows fit one chunk
#ifndef HS_TF_SUB_STRIDE
#define HS_TF_SUB_STRIDE 16
#endif
constexpr int kTfSubStride = HS_TF_SUB_STRIDE;
constexpr int kTfSubPasses = 2;
constexpr int64_t kTfSubMin = 32768;

struct TfState {
  double lo, hi, beta;      // bracket on beta = 1/T, point of the next sweep
  double dx, dx_old;        // last two step lengths (bisection safeguard)
  double nll, swept;        // mean NLL at the last swept beta, and that beta
  double T;                 // result
  long long used;           // rows entering the mean
  int lo_known, hi_known;   // g(lo) < 0 / g(hi) > 0 observed (else: clamp end not yet swept)
  int done, passes, converged;
  int newton_prev;          // the last move was a Newton step
  int mode;                 // 0: subsample warm-start sweeps, 1: first full sweep, 2: full sweeps
  int subpasses;
};

__device__ __forceinline__ uint32_t wordq(const uint4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}

// -inf for elements past C in the row's last 16-byte vector
template <bool BF16>
__device__ __forceinline__ uint4 tail_mask(const uint4& v, int tail) {
  uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    if (BF16) {
      const uint32_t lo = (2 * q < tail) ? (w[q] & 0xFFFFu) : 0xFF80u;
      const uint32_t hi = (2 * q + 1 < tail) ? (w[q] & 0xFFFF0000u) : 0xFF800000u;
      w[q] = lo | hi;
    } else if (q >= tail) {
      w[q] = kF32NegInf;
    }
  }
  return make_uint4(w[0], w[1], w[2], w[3]);
}

// Loads the group's chunk (vectors v0 + k*G + gl); slots past the row hold -inf.
// Loads the group's chunk (vectors v0 + k*G + gl); slots past the row hold -inf.
template <bool BF16, int G, int U>
__device__ __forceinline__ void load_chunk(uint4 (&v)[U], const uint4* rowp, int v0, int gl,
                                           int nvec, int tail, bool active) {
  const uint32_t f = BF16 ? kBf16NegInf2 : kF32NegInf;
#pragma unroll
  for (int k = 0; k < U; ++k) {
    const int vi = v0 + k * G + gl;
    if (active && vi < nvec) {
      v[k] = ldg_stream(rowp + vi);
      if (tail && vi == nvec - 1) v[k] = tail_mask<BF16>(v[k], tail);
    } else {
      v[k] = make_uint4(f, f, f, f);
    }
  }
}

// NaN-propagating max of a chunk, folded into m
template <bool BF16, int U>
__device__ __forceinline__ float chunk_max(const uint4 (&v)[U], float m) {
  if (BF16) {
    uint32_t mw = kBf16NegInf2;
#pragma unroll
    for (int k = 0; k < U; ++k) mw = bmax2(mw, bmax2(bmax2(v[k].x, v[k].y), bmax2(v[k].z, v[k].w)));
    return fmax_nan(m, fmax_nan(bf_lo(mw), bf_hi(mw)));
  }
#pragma unroll
  for (int k = 0; k < U; ++k)
    m = fmax_nan(m, fmax3_nan(__uint_as_float(v[k].x), __uint_as_float(v[k].y),
                              fmax_nan(__uint_as_float(v[k].z), __uint_as_float(v[k].w))));
  return m;
}

// s += e, w1 += e d, w2 += e d^2 over a chunk: d = x - m (exact), e = 2^{d c}
template <bool BF16, int U>
__device__ __forceinline__ void accum_chunk(const uint4 (&v)[U], f2_t m2, f2_t c2, uint32_t cw,
                                            float lowf, f2_t& s2, f2_t& w12, f2_t& w22) {
#pragma unroll
  for (int k = 0; k < U; ++k) {
#pragma unroll
    for (int q = 0; q < (BF16 ? 4 : 2); ++q) {
      f2_t x;
      if (BF16) {
        const uint32_t u = bmax2_plain(wordq(v[k], q), cw);
        x = f2(bf_lo(u), bf_hi(u));
      } else {
        x = f2(fmaxf(__uint_as_float(wordq(v[k], 2 * q)), lowf),
               fmaxf(__uint_as_float(wordq(v[k], 2 * q + 1)), lowf));
      }
      const f2_t d = f2sub(x, m2);
      const f2_t z = f2mul(d, c2);
      const f2_t e = f2(ex2(f2lo(z)), ex2(f2hi(z)));
      s2 = f2add(s2, e);
      const f2_t t = f2mul(e, d);
      w12 = f2add(w12, t);
      w22 = f2fma(t, d, w22);
    }
  }
}

// The group leader's verdict on a row with max m: used (valid, finite label
// logit) and dy = x_y - m.  Invalid rows (NaN / +inf / all -inf) flag status.
template <bool BF16>
__device__ __forceinline__ bool row_verdict(const TfArgs& a, float m, const uint4* rowp, int32_t lab,
                                            float* dy) {
  const bool valid = (m < INFINITY) && (m > -INFINITY);       // false for NaN too
  if (!valid && a.status) atomicOr(a.status, HS_STATUS_NONFINITE);
  float xy = -INFINITY;
  if (valid && lab >= 0 && (int64_t)lab < a.C) {
    if (BF16) {
      const unsigned short u = __ldg(reinterpret_cast<const unsigned short*>(rowp) + lab);
      xy = __uint_as_float((uint32_t)u << 16);
    } else {
      xy = __ldg(reinterpret_cast<const float*>(rowp) + lab);
    }
  }
  *dy = xy - m;
  return valid && xy > -INFINITY;
}

template <typename T, int G>
__device__ __forceinline__ T group_sum(T v) {
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// bf16x2 word L <= m - off with 2^{(L - m) c} < 2^-127 (flushed to 0 by
// ex2.approx.ftz): clamping x >= L leaves every non-zero term untouched and
// turns -inf (masked class) into a finite value, so e * d stays 0.  The
// offset is at least |m| * 2^-7 so that m - off is not absorbed by rounding.
__device__ __forceinline__ uint32_t clamp_word_bf16(float m, float c) {
  const float off = fmaxf(128.0f / c, fabsf(m) * 0.0078125f);
  const uint32_t u = (uint32_t)__bfloat16_as_ushort(__float2bfloat16_rd(m - off));
  return u | (u << 16);
}

// One safeguarded Newton update of a stage's state from the means at s.beta.
__device__ void tf_update(TfState& s, double nll, double g, double h, const TfArgs& a) {
  const double beta = s.beta;
  s.passes += 1;
  s.nll = nll;
  s.swept = beta;
  if (beta == a.blo0 && g >= 0.0) {        // NLL non-decreasing over the range: T = t_hi
    s.T = a.t_hi;
    s.done = s.converged = 1;
    return;
  }
  if (beta == a.bhi0 && g <= 0.0) {        // non-increasing: T = t_lo
    s.T = a.t_lo;
    s.done = s.converged = 1;
    return;
  }
  // g == 0 with h == 0: every used row is saturated in fp32 (all mass on the
  // label, the other terms below 2^-126); the true derivative is negative
  // there, so the point is treated as g < 0 (towards lower T)
  if (g == 0.0 && h > 0.0) {
    s.T = 1.0 / beta;
    s.done = s.converged = 1;
    return;
  }
  if (g > 0.0) {
    s.hi = beta;
    s.hi_known = 1;
  } else {
    s.lo = beta;
    s.lo_known = 1;
  }
  const double step = g / h;
  const double bn = beta - step;
  double next;
  if (h > 0.0 && isfinite(bn) && bn > s.lo && bn < s.hi && fabs(2.0 * step) <= s.dx_old) {
    if (fabs(step) <= a.tol * beta) {       // converged: report the Newton point
      s.T = 1.0 / bn;
      s.done = s.converged = 1;
      return;
    }
    // quadratic regime (two Newton steps in a row): the error left after this
    // step is ~ step^3 / prev_step^2; finish without a confirming sweep when it
    // is 10x below the tolerance
    if (s.newton_prev && s.dx > 0.0) {
      const double st = fabs(step);
      if (st * st * st <= 0.1 * a.tol * beta * s.dx * s.dx) {
        s.T = 1.0 / bn;
        s.done = s.converged = 1;
        return;
      }
    }
    next = bn;
  } else if (g > 0.0 && !s.lo_known && !(h > 0.0 && bn > s.lo)) {
    next = s.lo;                            // root may lie below the range: probe t_hi
  } else if (g <= 0.0 && !s.hi_known && !(h > 0.0 && bn < s.hi)) {
    next = s.hi;                            // probe t_lo
  } else {
    next = sqrt(s.lo * s.hi);               // geometric bisection of the bracket
  }
  if (s.lo_known && s.hi_known && (s.hi - s.lo) <= a.tol * s.lo) {
    s.T = 2.0 / (s.lo + s.hi);
    s.done = s.converged = 1;
    return;
  }
  s.newton_prev = next == bn ? 1 : 0;
  s.dx_old = s.dx;
  s.dx = fabs(next - beta);
  s.beta = next;
}

// Fixed-order sum over CTAs of partial[j][b][c], c < ncomp (identical in every CTA).
__device__ __forceinline__ void reduce_partials(const double* part, int nb, int ncta, double* red,
                                                const int* skip, int ncomp) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int p = warp; p < nb * kTfComp; p += kTfWarps) {
    const int b = p / kTfComp;
    if (skip[b] || p % kTfComp >= ncomp) continue;
    double v = 0.0;
    for (int j = lane; j < ncta; j += 32) v += __ldcg(part + ((size_t)j * nb + b) * kTfComp + (p % kTfComp));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
    if (lane == 0) red[p] = v;
  }
}

template <bool BF16, int G, int U>
__global__ void __launch_bounds__(kTfThreads, 1) temp_fit_kernel(const TfArgs a) {
  pdl_start();
  cg::grid_group grid = cg::this_grid();
  __shared__ TfState st[kMaxBatch];
  __shared__ double wacc[kTfWarps][kMaxBatch * kTfComp];
  __shared__ double red[kMaxBatch * kTfComp];
  __shared__ int skip[kMaxBatch];
  __shared__ int s_live[kMaxBatch], s_nl;
  __shared__ long long s_cum[kMaxBatch + 1];
  constexpr int GPW = 32 / G;
  constexpr int CH = G * U;                              // vectors per group per chunk
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int gl = lane & (G - 1), grp = lane / G;
  const int nb = a.nbatch;
  const int64_t n = a.n;
  const int64_t wstride = (int64_t)gridDim.x * kTfWarps * GPW;       // rows per warp step
  const int64_t wbase = ((int64_t)blockIdx.x * kTfWarps + warp) * GPW;
  double* part0 = a.partial;
  double* part1 = a.partial + (size_t)gridDim.x * nb * kTfComp;
  // rows of one chunk: the max / label / validity sweep is folded into the
  // first Newton sweep (the row is in registers for both)
  const bool fused = a.nvec <= CH;
  const float nanf_ = __int_as_float(0x7FC00000);

  if (threadIdx.x < nb) {
    TfState& s = st[threadIdx.x];
    s.lo = a.blo0;
    s.hi = a.bhi0;
    s.beta = fmin(fmax(1.0, a.blo0), a.bhi0);             // start at T = 1 (clamped)
    s.dx = s.dx_old = 2.0 * (a.bhi0 - a.blo0) + 1.0;
    s.nll = __longlong_as_double(0x7FF8000000000000ll);
    s.swept = s.nll;
    s.T = s.nll;
    s.used = -1;
    s.lo_known = s.hi_known = 0;
    s.newton_prev = 0;
    s.mode = !fused ? 2 : (n >= kTfSubMin ? 0 : 1);
    s.subpasses = 0;
    s.done = 0;
    s.passes = 0;
    s.converged = 0;
    skip[threadIdx.x] = 0;
  }

  if (!fused) {
    // ---- sweep 0: row max m (NaN-propagating), dy = x_y - m, validity
    for (int b = 0; b < nb; ++b) {
      const char* base = (const char*)a.bptr[b];
      double used = 0.0;
      for (int64_t r0 = wbase; r0 < n; r0 += wstride) {
        const int64_t row = r0 + grp;
        const bool active = row < n;
        const uint4* rowp = reinterpret_cast<const uint4*>(base + (active ? row : 0) * a.row_bytes);
        int32_t lab = 0;
        if (active && gl == 0) lab = __ldg(a.labels + row);
        float m = -INFINITY;
        for (int v0 = 0; v0 < a.nvec; v0 += CH) {
          uint4 v[U];
          load_chunk<BF16, G, U>(v, rowp, v0, gl, a.nvec, a.tail, active);
          m = chunk_max<BF16, U>(v, m);
        }
#pragma unroll
        for (int o = G / 2; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
        if (active && gl == 0) {
          float dy;
          const bool use = row_verdict<BF16>(a, m, rowp, lab, &dy);
          a.rowstat[(size_t)b * n + row] = use ? make_float2(m, dy) : make_float2(nanf_, 0.f);
          used += use ? 1.0 : 0.0;
        }
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) used += __shfl_xor_sync(0xFFFFFFFFu, used, o);
      if (lane == 0) wacc[warp][b * kTfComp] = used;
    }
    __syncthreads();
    if (threadIdx.x < nb) {
      double u = 0.0;
      for (int w = 0; w < kTfWarps; ++w) u += wacc[w][threadIdx.x * kTfComp];
      part0[((size_t)blockIdx.x * nb + threadIdx.x) * kTfComp] = u;
    }
    grid.sync();
    reduce_partials(part0, nb, gridDim.x, red, skip, 1);
    __syncthreads();
    if (threadIdx.x < nb) {
      st[threadIdx.x].used = (long long)red[threadIdx.x * kTfComp];
      st[threadIdx.x].done = st[threadIdx.x].used == 0;
    }
  }
  __syncthreads();

  // ---- Newton sweeps: one pass over the logits at st[b].beta per live stage.
  // The warp-rows (GPW rows) of all live stages form one list dealt round-robin
  // to the warps, so a pass is balanced to one warp-row across the grid; a
  // warp visits each stage in one contiguous run and flushes its sums when the
  // stage changes (warp-uniform).
  const int64_t gwarp = (int64_t)blockIdx.x * kTfWarps + warp;
  const int64_t nwarps = (int64_t)gridDim.x * kTfWarps;
  const int64_t nw = (n + GPW - 1) / GPW;                  // warp-rows per stage
  const int64_t n_sub = (n + kTfSubStride - 1) / kTfSubStride;
  const int64_t nw_sub = (n_sub + GPW - 1) / GPW;          // warp-rows of a subsample sweep
  for (int pass = 1; pass <= a.max_passes + kTfSubPasses; ++pass) {
    // the live stages and their warp-row offsets (identical in every thread; in
    // shared memory to keep the lookup out of registers / local memory)
    if (threadIdx.x == 0) {
      int k = 0;
      s_cum[0] = 0;
      for (int b = 0; b < nb; ++b)
        if (!st[b].done) {
          s_live[k] = b;
          s_cum[k + 1] = s_cum[k] + (st[b].mode == 0 ? nw_sub : nw);
          ++k;
        }
      s_nl = k;
    }
    __syncthreads();
    const int nl = s_nl;
    const int* live = s_live;
    const long long* cum = s_cum;
    if (nl == 0) break;
    double* part = (pass & 1) ? part1 : part0;
    int mode = 2;                                          // of the stage being swept
    if (lane < nb * kTfComp) wacc[warp][lane] = 0.0;     // stages this warp does not visit
    __syncwarp();
    int li = -1, b = -1;
    const char* base = nullptr;
    double beta = 0.0;
    float c = 0.f;
    f2_t c2 = 0;
    double acc_u = 0.0, acc_nll = 0.0, acc_g = 0.0, acc_h = 0.0;
    auto flush = [&]() {
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc_u += __shfl_xor_sync(0xFFFFFFFFu, acc_u, o);
        acc_nll += __shfl_xor_sync(0xFFFFFFFFu, acc_nll, o);
        acc_g += __shfl_xor_sync(0xFFFFFFFFu, acc_g, o);
        acc_h += __shfl_xor_sync(0xFFFFFFFFu, acc_h, o);
      }
      if (lane == 0) {
        wacc[warp][b * kTfComp + 0] = acc_u;
        wacc[warp][b * kTfComp + 1] = acc_nll;
        wacc[warp][b * kTfComp + 2] = acc_g;
        wacc[warp][b * kTfComp + 3] = acc_h;
      }
      acc_u = acc_nll = acc_g = acc_h = 0.0;
    };
    for (int64_t wr = gwarp; wr < cum[nl]; wr += nwarps) {
      int lj = li < 0 ? 0 : li;
      while (wr >= cum[lj + 1]) ++lj;                        // warp-uniform
      if (lj != li) {
        if (li >= 0) flush();
        li = lj;
        b = live[li];
        base = (const char*)a.bptr[b];
        beta = st[b].beta;
        c = (float)(beta * 1.4426950408889634);             // beta * log2(e)
        c2 = f2(c, c);
        mode = st[b].mode;
      }
      const bool first = mode <= 1;                         // m, dy from registers
      {
        const int64_t rl = (wr - cum[li]) * GPW + grp;
        const int64_t row = mode == 0 ? rl * kTfSubStride : rl;
        const bool inb = mode == 0 ? rl < n_sub : row < n;
        const uint4* rowp = reinterpret_cast<const uint4*>(base + (inb ? row : 0) * a.row_bytes);
        // the row's first chunk is loaded together with its row state (the
        // address does not depend on it)
        uint4 v[U];
        float2 rs = make_float2(nanf_, 0.f);
        int32_t lab = 0;
        if (first) {
          if (inb && gl == 0) lab = __ldg(a.labels + row);
        } else if (inb) {
          rs = __ldcg(a.rowstat + (size_t)b * n + row);
        }
        load_chunk<BF16, G, U>(v, rowp, 0, gl, a.nvec, a.tail, inb);
        if (first) {
          float m = chunk_max<BF16, U>(v, -INFINITY);
#pragma unroll
          for (int o = G / 2; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
          float dy = 0.f;
          bool use = false;
          if (inb && gl == 0) {
            use = row_verdict<BF16>(a, m, rowp, lab, &dy);
            if (mode == 1) a.rowstat[(size_t)b * n + row] = use ? make_float2(m, dy) : make_float2(nanf_, 0.f);
            acc_u += use ? 1.0 : 0.0;
          }
          const int leader = grp * G;
          use = __shfl_sync(0xFFFFFFFFu, use, leader);
          dy = __shfl_sync(0xFFFFFFFFu, dy, leader);
          rs = use ? make_float2(m, dy) : make_float2(nanf_, 0.f);
        }
        const bool active = rs.x == rs.x;                     // used row
        const float m = active ? rs.x : 0.f;
        const f2_t m2 = f2(m, m);
        const uint32_t cw = BF16 ? clamp_word_bf16(m, c) : 0u;
        const float lowf = m - fmaxf(128.0f / c, fabsf(m) * 0.0078125f);
        f2_t s2 = f2(0.f, 0.f), w12 = f2(0.f, 0.f), w22 = f2(0.f, 0.f);
        accum_chunk<BF16, U>(v, m2, c2, cw, lowf, s2, w12, w22);
        for (int v0 = CH; v0 < a.nvec; v0 += CH) {           // longer rows: further chunks
          load_chunk<BF16, G, U>(v, rowp, v0, gl, a.nvec, a.tail, inb && active);
          accum_chunk<BF16, U>(v, m2, c2, cw, lowf, s2, w12, w22);
        }
        float s = group_sum<float, G>(f2lo(s2) + f2hi(s2));
        float w1 = group_sum<float, G>(f2lo(w12) + f2hi(w12));
        float w2 = group_sum<float, G>(f2lo(w22) + f2hi(w22));
        if (active && gl == 0) {
          // per-row moments in fp32 (one MUFU.RCP; s in [1, C]), row sums in fp64:
          // g_i and h_i only steer the Newton iteration, whose stop (2^-21 in beta)
          // is far above their fp32 rounding; the fp64 divisions cost ~10 % of a
          // sweep's instructions on the warp's critical path
#ifdef HS_AB_TF_FP64_ROW
          const double ds = (double)s, mean = (double)w1 / ds;
          acc_nll += (double)logf(s) - beta * (double)rs.y;
          acc_g += mean - (double)rs.y;
          acc_h += fmax((double)w2 / ds - mean * mean, 0.0);
#else
          const float inv = __fdividef(1.0f, s), mean = w1 * inv;
          acc_nll += (double)logf(s) - beta * (double)rs.y;
          acc_g += (double)(mean - rs.y);
          acc_h += (double)fmaxf(fmaf(w2, inv, -mean * mean), 0.0f);
#endif
        }
      }
    }
    if (li >= 0) flush();
    __syncthreads();
    if (threadIdx.x < nb * kTfComp) {
      const int b = threadIdx.x / kTfComp;
      skip[b] = st[b].done;
      if (!st[b].done) {
        double v = 0.0;
        for (int w = 0; w < kTfWarps; ++w) v += wacc[w][threadIdx.x];
        part[(size_t)blockIdx.x * nb * kTfComp + threadIdx.x] = v;
      }
    }
    grid.sync();
    reduce_partials(part, nb, gridDim.x, red, skip, kTfComp);
    __syncthreads();
    if (threadIdx.x < nb && !st[threadIdx.x].done) {
      TfState& s = st[threadIdx.x];
      const double* r = red + threadIdx.x * kTfComp;
      if (s.mode == 0) {
        // warm start on the subsample: plain Newton, clamped to the range; no
        // convergence decision is taken on a sample
        const double u = r[0];
        double step = 0.0;
        if (u > 0.0) {
          const double g = r[2] / u, h = r[3] / u;
          step = (h > 0.0 && isfinite(g / h)) ? g / h : 0.0;
          s.beta = fmin(fmax(s.beta - step, a.blo0), a.bhi0);
        }
        if (u == 0.0 || ++s.subpasses >= kTfSubPasses || fabs(step) <= 1e-3 * s.beta) s.mode = 1;
      } else {
        if (s.mode == 1) s.used = (long long)r[0];
        s.mode = 2;
        if (s.used == 0) {
          s.done = 1;                                     // no usable row: T = NaN
        } else {
          const double inv = 1.0 / (double)s.used;
          tf_update(s, r[1] * inv, r[2] * inv, r[3] * inv, a);
          if (!s.done && s.passes >= a.max_passes) {      // full-sweep budget spent
            s.T = 1.0 / s.swept;
            s.done = 1;                                   // converged stays 0: flagged below
          }
        }
      }
    }
    __syncthreads();
  }

  if (blockIdx.x == 0 && threadIdx.x < nb) {
    TfState& s = st[threadIdx.x];
    if (!s.done && s.passes > 0) s.T = 1.0 / s.swept;   // (defensive) last swept point
    if (!s.converged && s.used > 0 && a.status) atomicOr(a.status, HS_STATUS_NOT_CONVERGED);
    a.T[threadIdx.x] = (float)s.T;
    if (a.nll) a.nll[threadIdx.x] = s.nll;
    if (a.passes) a.passes[threadIdx.x] = s.passes;
    if (a.used) a.used[threadIdx.x] = s.used < 0 ? 0 : s.used;
  }
}

template <bool BF16, int G, int U>
cudaError_t launch_tf(const TfArgs& a, cudaStream_t s) {
  auto kern = temp_fit_kernel<BF16, G, U>;
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kTfThreads, 0);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorLaunchOutOfResources;
  int grid = num_sms() * per_sm;
  if (grid > kTfMaxGrid) grid = kTfMaxGrid;
  TfArgs args = a;
  void* params[] = {(void*)&args};
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(kTfThreads);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = s;
  cudaLaunchAttribute at[2];
  at[0].id = cudaLaunchAttributeCooperative;
  at[0].val.cooperative = 1;
  at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[1].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 2 : 1;
  e = cudaLaunchKernelExC(&cfg, (const void*)kern, params);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

template <bool BF16>
cudaError_t launch_tf_dt(const TfArgs& a, cudaStream_t s) {
  // lanes per row: the row in one chunk of 4 vectors per lane where possible
  // (8 per lane at 16 lanes for 65..128 vectors: two rows per warp, 4 KB of
  // loads in flight per warp); longer rows stream 32 x 4-vector chunks
  const int nv = a.nvec;
  if (nv <= 8) return launch_tf<BF16, 2, 4>(a, s);
  if (nv <= 16) return launch_tf<BF16, 4, 4>(a, s);
  if (nv <= 32) return launch_tf<BF16, 8, 4>(a, s);
  if (nv <= 64) return launch_tf<BF16, 16, 4>(a, s);
  if (nv <= 128 && !getenv("HS_TF_G32")) return launch_tf<BF16, 16, 8>(a, s);
  return launch_tf<BF16, 32, 4>(a, s);
}

}  // namespace

size_t temp_fit_ws_bytes(int nbatch, int64_t n) {
  const size_t rows = (size_t)nbatch * (size_t)(n > 0 ? n : 0) * sizeof(float2);
  return (rows + 255) / 256 * 256 + (size_t)2 * kTfMaxGrid * nbatch * kTfComp * sizeof(double);
}

cudaError_t launch_temp_fit(TfArgs a, bool bf16, void* ws, cudaStream_t s) {
  const size_t rows = (size_t)a.nbatch * (size_t)a.n * sizeof(float2);
  a.rowstat = reinterpret_cast<float2*>(ws);
  a.partial = reinterpret_cast<double*>(reinterpret_cast<char*>(ws) + (rows + 255) / 256 * 256);
  return bf16 ? launch_tf_dt<true>(a, s) : launch_tf_dt<false>(a, s);
}

}  // namespace hs
