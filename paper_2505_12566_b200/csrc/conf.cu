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
// Launch shapes:
//   * conf_async_kernel -- G lanes per row, the row in registers, the next row
//     prefetched by per-lane cp.async into a per-warp shared-memory double
//     buffer (default for rows of <= 128 x 16 B: ViT/ImageNet classifiers).
//   * conf_warp_kernel  -- the same reduction with a register double buffer
//     (rows up to 512 x 16 B, e.g. C <= 4096 bf16 / 2048 fp32).  Exact
//     two-step (row max by shuffle, then exponentials) -- no online rescaling.
//   * conf_tma_kernel   -- the same with a TMA bulk-copy ring (selectable).
//   * conf_cta_kernel   -- one CTA per row, persistent over rows, per-thread
//     online (max, sum, weighted sum) over 8-vector chunks, block merge
//     (vocabulary-sized rows: T5 32,128, Llama 128,256).
#include <cooperative_groups.h>
#include <cuda_bf16.h>
#include <cstdlib>
#include <cstring>

#include "hs_common.cuh"
#include "hs_internal.h"

namespace hs {

namespace {

struct RowOut {
  float m;     // raw row max (NaN / +inf / -inf => invalid row)
  float s;     // sum 2^a
  float w;     // sum 2^a * a
  uint32_t am; // argmax
  float e0;    // 2^a of the max element (1 when a is formed as (x - m) * c)
};

// `lab`: the row's label, loaded by the caller ahead of time (a.labels only)
__device__ __forceinline__ float write_row(const ConfArgs& a, int64_t row, int32_t lab,
                                           const RowOut& r) {
  const bool bad = !(r.m < INFINITY) || (r.m == -INFINITY);
  float c;
  int32_t am = (int32_t)r.am;
  if (bad) {
    c = __int_as_float(0x7FC00000);
    am = -1;
    if (a.status) atomicOr(a.status, HS_STATUS_NONFINITE);
  } else {
    const float p = __fdividef(r.e0, r.s);   // s in [1, C]: MUFU.RCP + FMUL, <= 2 ulp
    if (a.kind == HS_CONF_MAXPROB_SQ) {
      c = p * p;
    } else if (a.kind == HS_CONF_ENTROPY) {
      // exp(-H) = 2^{w/s - log2 s} (invariant to a common shift of every a);
      // full-precision exp2f/log2f
      c = exp2f(r.w / r.s - log2f(r.s));
    } else {
      c = p;
    }
  }
  a.conf[row] = c;
  if (a.conf2) a.conf2[row] = bad ? __int_as_float(0x7FC00000) : exp2f(r.w / r.s - log2f(r.s));
  if (a.argmax) a.argmax[row] = am;
  if (a.ok) a.ok[row] = (uint8_t)(a.labels ? (!bad && lab == am) : 0);
  if (a.last_ids_out) a.last_ids_out[row] = a.last_ids ? a.last_ids[row] : row;
  return c;
}


__device__ __forceinline__ int64_t live_rows(const ConfArgs& a) {
  int64_t n = a.n;
  if (a.d_n) {
    int64_t dn = *a.d_n;
    n = dn < n ? dn : n;
  }
  return n * a.L * (int64_t)a.nbatch;
}

// last stage (ConfArgs::last_counts): every live row is accepted
__device__ __forceinline__ void write_last_counts(const ConfArgs& a) {
  if (a.last_counts && blockIdx.x == 0 && threadIdx.x == 0) {
    a.last_counts[0] = live_rows(a);
    a.last_counts[1] = 0;
  }
}

__device__ __forceinline__ uint32_t word(const uint4& v, int q) {
  return q == 0 ? v.x : q == 1 ? v.y : q == 2 ? v.z : v.w;
}

// Where output row `row` reads its logits: batch base pointer, temperature
// factor and source row (row_index applies within the batch).
struct RowSrc {
  const char* base;
  float c;
  int64_t src;
};
__device__ __forceinline__ int64_t batch_local(const ConfArgs& a, int64_t row, int* b) {
  *b = 0;
  if (a.nbatch > 1) {
    // rows < 2^32: multiply by the host-computed reciprocal (no integer divide)
    *b = a.bmagic ? (int)__umul64hi((uint64_t)row, a.bmagic) : (int)row;
    return row - (int64_t)(*b) * a.brows;
  }
  return row;
}
// The gathered-row lookup (row_index) of `row`, issued ahead of its use so the
// dependent logits loads of a later iteration do not wait on it.
__device__ __forceinline__ int64_t fetch_index(const ConfArgs& a, int64_t row) {
  if (!a.row_index) return 0;
  int b;
  const int64_t local = batch_local(a, row, &b);
  return a.L == 1 ? a.row_index[local] : a.row_index[local / a.L];
}
template <bool RIDX>
__device__ __forceinline__ int64_t fetch_index_t(const ConfArgs& a, int64_t row) {
  if constexpr (!RIDX) return 0;
  else return fetch_index(a, row);
}
__device__ __forceinline__ RowSrc locate_with(const ConfArgs& a, int64_t row, int64_t fetched) {
  int b;
  const int64_t local = batch_local(a, row, &b);
  RowSrc r{(const char*)a.logits, a.c, local};
  if (a.nbatch > 1) {
    r.base = (const char*)a.bptr[b];
    r.c = a.bc[b];
  }
  if (a.row_index) r.src = a.L == 1 ? fetched : fetched * a.L + local % a.L;
  return r;
}
// Batched launches: the rows of one group only increase, so the group keeps
// the bounds of its current batch and re-derives them only when a row leaves
// them (at most nbatch - 1 times, plus the clamped rows of inactive groups).
struct BatchCur {
  uint32_t start, end;     // batched rows < 2^32
  const char* base;
  float c;
};
__device__ __forceinline__ BatchCur cur_init(const ConfArgs& a) {
  return BatchCur{0u, a.nbatch > 1 ? 0u : 0xFFFFFFFFu, (const char*)a.logits, a.c};
}
template <bool RIDX = true>
__device__ __forceinline__ RowSrc locate_cur(const ConfArgs& a, BatchCur& k, int64_t row,
                                             int64_t fetched) {
  if ((uint32_t)row < k.start || (uint32_t)row >= k.end) {
    int b;
    const int64_t local = batch_local(a, row, &b);
    k.start = (uint32_t)(row - local);
    k.end = k.start + (uint32_t)a.brows;
    k.base = (const char*)a.bptr[b];
    k.c = a.bc[b];
  }
  const int64_t local = row - (int64_t)k.start;
  RowSrc r{k.base, k.c, local};
  if (RIDX && a.row_index) r.src = a.L == 1 ? fetched : fetched * a.L + local % a.L;
  return r;
}
__device__ __forceinline__ RowSrc locate(const ConfArgs& a, int64_t row) {
  return locate_with(a, row, fetch_index(a, row));
}
// the label of a located row, issued with its logits loads (used at write time)
__device__ __forceinline__ int32_t fetch_label(const ConfArgs& a, const RowSrc& r) {
  return a.labels ? __ldg(a.labels + r.src) : 0;
}

// -inf for the out-of-row elements of the last partial 16-byte vector
// (value semantics only: no address is taken, so nothing spills to local memory)
template <bool BF16>
__device__ __forceinline__ uint32_t mask_word(uint32_t w, int q, int tail) {
  if (BF16) {
    const uint32_t lo = (2 * q < tail) ? (w & 0xFFFFu) : 0xFF80u;
    const uint32_t hi = (2 * q + 1 < tail) ? (w & 0xFFFF0000u) : 0xFF800000u;
    return lo | hi;
  }
  return (q < tail) ? w : kF32NegInf;
}
template <bool BF16>
__device__ __forceinline__ uint4 masked(const uint4& v, int tail) {
  return make_uint4(mask_word<BF16>(v.x, 0, tail), mask_word<BF16>(v.y, 1, tail),
                    mask_word<BF16>(v.z, 2, tail), mask_word<BF16>(v.w, 3, tail));
}

template <bool BF16>
__device__ __forceinline__ uint4 load_vec(const uint4* p, int vi, int nvec, int tail) {
  uint4 v;
  if (vi < nvec) {
    v = ldg_stream(p + vi);
    if (tail && vi == nvec - 1) v = masked<BF16>(v, tail);
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
  int r = BF16 ? 8 : 4;
#pragma unroll
  for (int q = 3; q >= 0; --q) {
    const uint32_t w = word(v, q);
    if (BF16) {
      if (bf_hi(w) == m) r = 2 * q + 1;
      if (bf_lo(w) == m) r = 2 * q;
    } else {
      if (__uint_as_float(w) == m) r = q;
    }
  }
  return r;
}

// Accumulate 2^a and 2^a * a of one vector into the packed accumulators.
template <bool BF16, bool ENTROPY>
__device__ __forceinline__ void vec_accum(const uint4& v, f2_t m2, f2_t c2, uint32_t clampw,
                                          f2_t& s2, f2_t& w2) {
  if (BF16) {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      uint32_t u = ENTROPY ? bmax2_plain(word(v, q), clampw) : word(v, q);
      f2_t a = f2mul(f2sub(f2(bf_lo(u), bf_hi(u)), m2), c2);
      f2_t e = f2(ex2(f2lo(a)), ex2(f2hi(a)));
      s2 = f2add(s2, e);
      if (ENTROPY) w2 = f2fma(e, a, w2);
    }
  } else {
#pragma unroll
    for (int q = 0; q < 2; ++q) {
      f2_t a = f2mul(f2sub(f2(__uint_as_float(word(v, 2 * q)), __uint_as_float(word(v, 2 * q + 1))), m2), c2);
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
// K1a: G lanes per row (a warp reduces 32/G rows at once), row in registers.
// Lane j of a group holds the row's 16-byte vectors j, j+G, j+2G, ... (NV of
// them), so one warp instruction advances 32/G rows and the per-row costs
// (shuffle trees, argmax, output) are amortised over G*NV*VE elements/lane.
// ---------------------------------------------------------------------------
// NaN-propagating max of one vector kept as a bf16x2 word (bf16) or fp32
template <bool BF16>
__device__ __forceinline__ uint32_t vec_maxw(const uint4& v) {
  if (BF16) return bmax2(bmax2(v.x, v.y), bmax2(v.z, v.w));
  return __float_as_uint(fmax3_nan(__uint_as_float(v.x), __uint_as_float(v.y),
                                   fmax_nan(__uint_as_float(v.z), __uint_as_float(v.w))));
}
// does the vector whose max word is w contain the value m?  Compared in fp32:
// IEEE equality (+0 == -0) with subnormals intact (a packed bf16x2 compare
// flushes subnormals and would misplace the argmax of tiny logits).
template <bool BF16>
__device__ __forceinline__ bool maxw_has(uint32_t w, float m) {
  if (BF16) return fmax_nan(bf_lo(w), bf_hi(w)) == m;
  return __uint_as_float(w) == m;
}

template <bool BF16, int NV, int G>
__device__ __forceinline__ void group_mask_tail(uint4 (&v)[NV], int gl, int nvec, int tail) {
  const int last = nvec - 1;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const bool p = (k * G + gl) == last;
    const uint4 m = masked<BF16>(v[k], tail);
    v[k] = make_uint4(p ? m.x : v[k].x, p ? m.y : v[k].y, p ? m.z : v[k].z, p ? m.w : v[k].w);
  }
}

// first element of the bf16 vector x equal to the NORMAL bf16 value whose
// bits are mb2 = (mb, mb): packed compare (exact for normal m; a subnormal
// element would be flushed to 0 != m)
__device__ __forceinline__ int vec_first_eq_bf16n(const uint4& x, uint32_t mb2) {
  int r = 8;
#pragma unroll
  for (int q = 3; q >= 0; --q) {
    asm("{\n\t.reg .pred p, h;\n\t"
        "setp.eq.bf16x2 p|h, %1, %2;\n\t"
        "@h mov.s32 %0, %3;\n\t"
        "@p mov.s32 %0, %4;\n\t}"
        : "+r"(r)
        : "r"(word(x, q)), "r"(mb2), "r"(2 * q + 1), "r"(2 * q));
  }
  return r;
}

// does the packed bf16x2 word w hold the NORMAL bf16 value whose bits are
// mb2 = (mb, mb) in either half?  (one packed compare; exact for normal m)
__device__ __forceinline__ bool bf2_has(uint32_t w, uint32_t mb2) {
  uint32_t r;
  asm("{\n\t.reg .pred p, h;\n\t"
      "setp.eq.bf16x2 p|h, %1, %2;\n\t"
      "or.pred p, p, h;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"(w), "r"(mb2));
  return r != 0u;
}

// Lowest k in [0, 8) whose vector max vmw[k] holds m (some vmw[k] does): a
// descent of the pairwise max tree -- 3 packed compares and 4 selects instead
// of one compare and two selects per vector.
__device__ __forceinline__ int tree_first8(const uint32_t (&v)[8], uint32_t mb2) {
  const uint32_t p0 = bmax2(v[0], v[1]), p2 = bmax2(v[4], v[5]);
  const uint32_t q0 = bmax2(p0, bmax2(v[2], v[3]));
  const bool l1 = bf2_has(q0, mb2);                 // in vectors 0..3?
  const bool l2 = bf2_has(l1 ? p0 : p2, mb2);        // in the first pair of that half?
  const uint32_t w = l1 ? (l2 ? v[0] : v[2]) : (l2 ? v[4] : v[6]);
  const bool l3 = bf2_has(w, mb2);                  // in the first vector of that pair?
  return (l1 ? 0 : 4) + (l2 ? 0 : 2) + (l3 ? 0 : 1);
}

// Returns the row's confidence on its group's lane 0 (0 on the other lanes and
// for an inactive group).
template <bool BF16, bool ENTROPY, int NV, int G>
__device__ __forceinline__ float group_reduce_row(const ConfArgs& a, const uint4 (&v)[NV],
                                                  bool active, int64_t row, int gl,
                                                  float c, const uint4* rowp, int32_t lab) {
  constexpr int VE = BF16 ? 8 : 4;
  const f2_t c2 = f2(c, c);
  // 1. row max (exact, NaN-propagating): packed per-vector maxima, then the group
  uint32_t vmw[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) vmw[k] = vec_maxw<BF16>(v[k]);
  uint32_t lw;
  if constexpr (BF16 && NV == 8) {   // pairwise tree: shared with the argmax descent
    lw = bmax2(bmax2(bmax2(vmw[0], vmw[1]), bmax2(vmw[2], vmw[3])),
               bmax2(bmax2(vmw[4], vmw[5]), bmax2(vmw[6], vmw[7])));
  } else {
    lw = vmw[0];
#pragma unroll
    for (int k = 1; k < NV; ++k)
      lw = BF16 ? bmax2(lw, vmw[k]) : __float_as_uint(fmax_nan(__uint_as_float(lw), __uint_as_float(vmw[k])));
  }
  float m = BF16 ? fmax_nan(bf_lo(lw), bf_hi(lw)) : __uint_as_float(lw);
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));

  // 2. argmax = lowest index holding m.  (i) each lane: lowest of its vectors
  //    whose packed max contains m -- bf16: one packed compare of the lane max,
  //    then a descent of the max tree (log2 NV compares); (ii) group min -> vector
  //    vi; (iii) the group re-reads that one 16-byte vector (an L2 hit: the row
  //    was just streamed) and finds the first element equal to m after the
  //    exponential pass has hidden the load.
  //    A zero/subnormal m (or fp32) takes the exact fp32 compares.
#ifdef HS_EXP_NOARGMAX
  const unsigned am = 0;
#else
  unsigned vi = 0xFFFFFFFFu;
  // zero / subnormal row max (rare): packed compares would flush; exact path
  const bool slow = BF16 && (m == m) && !(fabsf(m) >= 1.17549435e-38f);
  const bool anyslow = BF16 && __any_sync(0xFFFFFFFFu, slow);
  const uint32_t mb2 = (__float_as_uint(m) >> 16) * 0x10001u;
  if (BF16) {
#ifndef HS_AB_LINEAR_ARGMAX
    if constexpr (NV == 8) {
      if (bf2_has(lw, mb2)) vi = (unsigned)(tree_first8(vmw, mb2) * G + gl);
    } else
#endif
    {
#pragma unroll
      for (int k = NV - 1; k >= 0; --k)
        if (bf2_has(vmw[k], mb2)) vi = (unsigned)(k * G + gl);
    }
  } else {
#pragma unroll
    for (int k = NV - 1; k >= 0; --k)
      if (__uint_as_float(vmw[k]) == m) vi = (unsigned)(k * G + gl);
  }
  if (anyslow) {
    if (slow) {
      vi = 0xFFFFFFFFu;
#pragma unroll
      for (int k = NV - 1; k >= 0; --k)
        if (maxw_has<BF16>(vmw[k], m)) vi = (unsigned)(k * G + gl);
    }
  }
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) vi = min(vi, (unsigned)__shfl_xor_sync(0xFFFFFFFFu, vi, o));
  // every lane of the group reads the same vector (one broadcast transaction);
  // an invalid row (no match) reads vector 0 and is discarded by write_row
  // (A/B: reading it from the shared-memory stage instead, behind a
  // __syncwarp, was 4 % slower than this L2 hit)
  const uint4 xv = __ldg(rowp + (vi < (unsigned)a.nvec ? vi : 0u));
#endif

  // 3. exponentials with the common max: a = (x - m) * c, x - m formed exactly
  //    (FADD2, then FMUL2: one rounding, so the 1e-5 tolerance holds at T = 0.05)
  f2_t s2 = f2(0.f, 0.f), w2 = f2(0.f, 0.f);
  const bool valid = (m < INFINITY) && (m > -INFINITY);
#ifdef HS_EXP_NOEXP
  if (valid) s2 = f2(1.f, 0.f);
  if (false) {
#else
  {   // unconditional: an invalid row's sums are discarded by write_row
#endif
    const uint32_t cw = ENTROPY && BF16 ? entropy_clamp_word(m, c) : 0u;
    const f2_t m2 = f2(m, m);
#pragma unroll
    for (int k = 0; k < NV; ++k) vec_accum<BF16, ENTROPY>(v[k], m2, c2, cw, s2, w2);
  }
  float s = f2lo(s2) + f2hi(s2);
  float w = ENTROPY ? f2lo(w2) + f2hi(w2) : 0.f;
#pragma unroll
  for (int o = G / 2; o > 0; o >>= 1) {
    s += __shfl_xor_sync(0xFFFFFFFFu, s, o);
    if (ENTROPY) w += __shfl_xor_sync(0xFFFFFFFFu, w, o);
  }
#ifndef HS_EXP_NOARGMAX
  int e = BF16 ? vec_first_eq_bf16n(xv, mb2) : vec_first_eq<false>(xv, m);
  if (anyslow) {
    if (slow) e = vec_first_eq<true>(xv, m);
  }
  const unsigned am = vi * VE + (unsigned)e;
#endif
  float conf = 0.f;
  if (active && gl == 0) {
    RowOut r{m, s, w, am, 1.0f};
    conf = write_row(a, row, lab, r);
  }
  return conf;
}

template <bool L1>
__device__ __forceinline__ int64_t src_row(const ConfArgs& a, int64_t r) {
  if (!a.row_index) return r;
  if (L1) return a.row_index[r];
  return a.row_index[r / a.L] * a.L + r % a.L;
}

// 16-byte loads of one group's row, all issued back to back.  The pointer of
// an inactive group is clamped to a valid row, so every vector below nvec can
// be loaded unconditionally; only vector slots >= nvec need a default (-inf).
// FULL: (NV-1)*G <= nvec, i.e. only the last slot k = NV-1 can be out of range
// (no per-register default moves on the other NV-1 vectors).
template <bool BF16, int NV, int G, bool FULL>
__device__ __forceinline__ void group_load_row(uint4 (&v)[NV], const uint4* p, int gl, int nvec) {
  const uint32_t f = BF16 ? kBf16NegInf2 : kF32NegInf;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = k * G + gl;
    if (FULL && k < NV - 1) {
      v[k] = ldg_stream(p + vi);
    } else {
      uint4 r = make_uint4(f, f, f, f);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %4, %5;\n\t"
          "@p ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%6];\n\t}"
          : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
          : "r"(vi), "r"(nvec), "l"(p + vi));
      v[k] = r;
    }
  }
}

// LDG variant: ping-pong register buffers, the next rows' loads are issued
// before the current rows are reduced.
// Lanes holding <= 8 vectors (x2 for the prefetch) fit 128 registers: two CTAs
// (16 warps) per SM.  A/B: +3.5 % over 8 lanes x 16 vectors at one CTA per SM.
template <bool BF16, bool ENTROPY, int NV, int G, bool FULL>
__global__ void __launch_bounds__(256, (NV <= 8 ? 2 : 1)) conf_warp_kernel(const ConfArgs a) {
  pdl_start();
  write_last_counts(a);
  constexpr int RPW = 32 / G;      // rows per warp
  const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G;
  const int64_t stride = (((int64_t)gridDim.x * blockDim.x) >> 5) * RPW;
  const int64_t rows = live_rows(a);
  const int nvec = a.nvec;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (w0 * RPW >= rows) return;
  // Three-deep pipeline per group: row indices two rows ahead, logits one row
  // ahead (registers B), the current row (registers A) being reduced.  One
  // reduce site, B copied into A each pass (A/B: +1.5-5 % over two sites).
  uint4 A[NV], B[NV];
  int64_t rowA = w0 * RPW + grp;
  bool actA = rowA < rows;
  RowSrc rA = locate(a, actA ? rowA : 0), rB = rA;   // inactive groups read a valid row
  group_load_row<BF16, NV, G, FULL>(A, reinterpret_cast<const uint4*>(rA.base + rA.src * a.row_bytes),
                                    gl, nvec);
  int32_t labA = fetch_label(a, rA), labB = 0;
  int64_t rowB = rowA + stride;
  int64_t fB = fetch_index(a, rowB < rows ? rowB : 0);
  while (true) {
    const bool anyB = (rowB - grp) < rows;
    const bool actB = rowB < rows;
    const int64_t rowC = rowB + stride;
    int64_t fC = 0;
    if (anyB) {
      rB = locate_with(a, actB ? rowB : 0, actB ? fB : fetch_index(a, 0));
      group_load_row<BF16, NV, G, FULL>(B, reinterpret_cast<const uint4*>(rB.base + rB.src * a.row_bytes),
                                        gl, nvec);
      labB = fetch_label(a, rB);
      fC = fetch_index(a, rowC < rows ? rowC : 0);
    }
    if (a.tail) group_mask_tail<BF16, NV, G>(A, gl, nvec, a.tail);
    group_reduce_row<BF16, ENTROPY, NV, G>(a, A, actA, rowA, gl, rA.c,
                                           reinterpret_cast<const uint4*>(rA.base + rA.src * a.row_bytes),
                                           labA);
    if (!anyB) break;
#pragma unroll
    for (int k = 0; k < NV; ++k) A[k] = B[k];
    rowA = rowB;
    actA = actB;
    rA = rB;
    labA = labB;
    rowB = rowC;
    fB = fC;
  }
}

// ---------------------------------------------------------------------------
// K1c (NEXT-2): Top-K restricted confidence (reading G4): the
// softmax over the K largest logits of the row, K <= 32.  One warp per row,
// streaming the row in chunks of 32 lanes x 4 vectors (next chunk in flight).
// No exponential per element: per 16-byte vector the packed NaN-propagating
// max, the lane's running max / first vector (argmax), and one exact fp32
// compare of the vector max against wt, a lower bound of the row's K-th
// largest value.  A lane whose vector has elements > wt appends them to its
// own shared-memory column (no warp vote per element); at the end of a chunk,
// if some column may overflow, and at the end of the row, the columns are
// merged into the warp's top-K list (lane j = entry j) by K max-extractions
// (redux.sync over the lanes' current candidate maxima; only the owner lane
// rescans its column).
//   Seed: wt = K-th largest of the 32 lane maxima of the first chunk and the
//   list = K copies of wt.  Invariant: top-K(row) = top-K(list U elements >
//   wt seen later) -- at least K elements are >= wt, so elements <= wt can be
//   replaced by copies of wt.  Exact for ties (multisets of values).
// ---------------------------------------------------------------------------
#ifndef HS_TOPK_U
#define HS_TOPK_U 4
#endif
constexpr int kTopkU = HS_TOPK_U;          // vectors per lane per chunk
#ifndef HS_TOPK_SLACK
#define HS_TOPK_SLACK 8
#endif
constexpr int kTopkPB = 8 * kTopkU + HS_TOPK_SLACK;   // candidate slots per lane (>= one chunk's elements + slack)

__device__ __forceinline__ uint32_t f_order(float f) {   // monotone float -> u32
  const uint32_t u = __float_as_uint(f);
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float f_unorder(uint32_t k) {
  return __uint_as_float((k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k);
}
template <bool BF16>
__device__ __forceinline__ float elem(const uint4& v, int e) {
  const uint32_t w = word(v, BF16 ? e >> 1 : e);
  if (BF16) return (e & 1) ? bf_hi(w) : bf_lo(w);
  return __uint_as_float(w);
}

// new list = the K largest of {list} U {column of lane l: col[0..pn_l)}
// (col[i] = slot i of this lane; stride 32 floats between slots)
__device__ __noinline__ float topk_merge(float lst, float* col, int pn, int K, int lane) {
  float lmax = lane < K ? lst : -INFINITY;   // this lane's best remaining value
  int src = -1;                              // -1: the list entry, i: col[i]
  for (int i = 0; i < pn; ++i) {
    const float v = col[i * 32];
    if (v > lmax) { lmax = v; src = i; }
  }
  bool used_list = lane >= K;
  float out = -INFINITY;
  for (int j = 0; j < K; ++j) {
    const uint32_t key = f_order(lmax);
    const uint32_t mk = __reduce_max_sync(0xFFFFFFFFu, key);
    const unsigned bal = __ballot_sync(0xFFFFFFFFu, key == mk);
    if (lane == j) out = f_unorder(mk);
    if (lane == __ffs(bal) - 1) {            // consume it, rescan this lane
      if (src < 0) used_list = true;
      else col[src * 32] = -INFINITY;
      lmax = used_list ? -INFINITY : lst;
      src = -1;
      for (int i = 0; i < pn; ++i) {
        const float v = col[i * 32];
        if (v > lmax) { lmax = v; src = i; }
      }
    }
  }
  return out;
}

template <bool BF16, bool ENTROPY>
__global__ void __launch_bounds__(256, kTopkU <= 4 ? 3 : 2) conf_topk_kernel(const ConfArgs a) {
  pdl_start();
  write_last_counts(a);
  constexpr int VE = BF16 ? 8 : 4, U = kTopkU;
  extern __shared__ __align__(16) float s_col[];          // [8 warps][kTopkPB][32 lanes]
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  float* col = s_col + (size_t)warp * kTopkPB * 32 + lane;
  const int64_t rows = live_rows(a);
  const int nvec = a.nvec, K = a.top_k;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint32_t ninf = BF16 ? kBf16NegInf2 : kF32NegInf;
  for (int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; row < rows; row += nwarps) {
    const RowSrc r = locate(a, row);
    const uint4* p = reinterpret_cast<const uint4*>(r.base + r.src * a.row_bytes);
    const int32_t lab = fetch_label(a, r);
    uint4 x[U], y[U];
    uint32_t mw = ninf;                   // NaN-propagating packed lane max
    // argmax bookkeeping.  bf16: the first vector where the lo / hi half of the
    // lane's packed max rose (one packed compare per vector; exact whenever the
    // row max is a normal number -- zero/subnormal maxima are re-scanned below).
    // fp32: the lane's exact max and its first vector.
    int bv_lo = 0x7FFFFFFF, bv_hi = 0x7FFFFFFF;
    float best = -INFINITY;
    int bestv = 0x7FFFFFFF;
    float lst = -INFINITY, wt = -INFINITY;
    int pn = 0;                           // this lane's buffered candidates
    // one chunk: vectors v0 + u*32 + lane of this lane, in registers `c`
    auto chunk = [&](uint4 (&c)[U], int v0) {
      if (a.tail) {
#pragma unroll
        for (int u = 0; u < U; ++u)
          if (v0 + u * 32 + lane == nvec - 1) c[u] = masked<BF16>(c[u], a.tail);
      }
      uint32_t cw = ninf;                 // packed max of this lane's chunk
      uint32_t wv[U];                     // packed max of each vector
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t w = vec_maxw<BF16>(c[u]);
        wv[u] = w;
        const int vi = v0 + u * 32 + lane;
        if (BF16) {
          asm("{\n\t.reg .pred p, h;\n\t"
              "setp.gt.bf16x2 p|h, %2, %3;\n\t"
              "@p mov.s32 %0, %4;\n\t"
              "@h mov.s32 %1, %4;\n\t}"
              : "+r"(bv_lo), "+r"(bv_hi)
              : "r"(w), "r"(mw), "r"(vi));
          mw = bmax2(mw, w);
          cw = bmax2(cw, w);
        } else {
          const float f = __uint_as_float(w);
          mw = __float_as_uint(fmax_nan(__uint_as_float(mw), f));
          cw = __float_as_uint(fmaxf(__uint_as_float(cw), f));
          if (f > best) {
            best = f;
            bestv = vi;
          }
        }
      }
      const float lmx = BF16 ? fmaxf(bf_lo(cw), bf_hi(cw)) : __uint_as_float(cw);
      if (v0 == 0) {
        // seed: wt = K-th largest lane max of the first chunk, list = K copies
        uint32_t key = f_order(lmx);
        for (int j = 0; j < K; ++j) {
          const uint32_t mk = __reduce_max_sync(0xFFFFFFFFu, key);
          wt = f_unorder(mk);
          const unsigned bal = __ballot_sync(0xFFFFFFFFu, key == mk);
          if (lane == __ffs(bal) - 1) key = 0u;        // below every float key
        }
        lst = wt;
      }
#ifdef HS_EXP_TOPK_NOCAND
      if (false) {                        // timing experiment only: no candidates (wrong results)
#else
      if (lmx > wt) {                     // rare: append this lane's elements > wt
#endif
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const float vm = BF16 ? fmaxf(bf_lo(wv[u]), bf_hi(wv[u])) : __uint_as_float(wv[u]);
          if (vm > wt) {                  // only the vectors that hold one
#pragma unroll
            for (int e = 0; e < VE; ++e) {
              const float val = elem<BF16>(c[u], e);
              if (val > wt) col[32 * pn++] = val;
            }
          }
        }
      }
      // merge as soon as K candidates are buffered (raises wt early, so later
      // chunks rarely have any) or when a column could overflow in the next chunk
#ifndef HS_TOPK_MERGE_AT
#define HS_TOPK_MERGE_AT 8     // merge once 8K candidates are buffered (A/B: 1 -> 0.72, 4 -> 0.80, 8 -> 0.80 of peak, fastest step)
#endif
      if (__reduce_add_sync(0xFFFFFFFFu, (unsigned)pn) >= (unsigned)(HS_TOPK_MERGE_AT * K) ||
          __any_sync(0xFFFFFFFFu, pn > kTopkPB - 8 * kTopkU)) {
        __syncwarp();
        lst = topk_merge(lst, col, pn, K, lane);
        wt = __shfl_sync(0xFFFFFFFFu, lst, K - 1);
        pn = 0;
        __syncwarp();
      }
    };
    auto load = [&](uint4 (&c)[U], int v0) {
      if (v0 + 32 * U <= nvec) {          // full chunk: unconditional loads
#pragma unroll
        for (int u = 0; u < U; ++u) c[u] = ldg_stream(p + v0 + u * 32 + lane);
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u) {
          const int vi = v0 + u * 32 + lane;
          c[u] = vi < nvec ? ldg_stream(p + vi) : make_uint4(ninf, ninf, ninf, ninf);
        }
      }
    };
    // ping-pong: the next chunk's loads are issued before the current chunk
    load(x, 0);
    for (int v0 = 0;; v0 += 64 * U) {
      load(y, v0 + 32 * U);
      chunk(x, v0);
      if (v0 + 32 * U >= nvec) break;
      load(x, v0 + 64 * U);
      chunk(y, v0 + 32 * U);
      if (v0 + 64 * U >= nvec) break;
    }
    __syncwarp();
    if (__any_sync(0xFFFFFFFFu, pn > 0)) lst = topk_merge(lst, col, pn, K, lane);
    __syncwarp();
    // row statistics over the K list entries (m = the row max = entry 0)
    float m = BF16 ? fmax_nan(bf_lo(mw), bf_hi(mw)) : __uint_as_float(mw);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = fmax_nan(m, __shfl_xor_sync(0xFFFFFFFFu, m, o));
    const float c = r.c;
    float e = 0.f, ea = 0.f;
    if (lane < K && lst > -INFINITY) {
      const float av = (lst - m) * c;
      e = ex2(av);
      ea = e * av;
    }
    const float s = warp_sum(e);
    const float w = ENTROPY ? warp_sum(ea) : 0.f;
    // argmax: lowest vector holding m, then its first element (exact fp32)
    unsigned vi;
    if (BF16) {
      const float lo = bf_lo(mw), hi = bf_hi(mw);
      const int fv = lo > hi ? bv_lo : hi > lo ? bv_hi : min(bv_lo, bv_hi);
      vi = (fmaxf(lo, hi) == m) ? (unsigned)fv : 0xFFFFFFFFu;
      vi = __reduce_min_sync(0xFFFFFFFFu, vi);
      if (__any_sync(0xFFFFFFFFu, m == m && !(fabsf(m) >= 1.17549435e-38f))) {
        // zero / subnormal row max: the packed compares flushed; exact re-scan
        unsigned f = 0xFFFFFFFFu;
        for (int v = lane; v < nvec; v += 32) {
          uint4 q = __ldg(p + v);
          if (a.tail && v == nvec - 1) q = masked<BF16>(q, a.tail);
          if (maxw_has<BF16>(vec_maxw<BF16>(q), m)) { f = (unsigned)v; break; }
        }
        vi = __reduce_min_sync(0xFFFFFFFFu, f);
      }
    } else {
      vi = (best == m) ? (unsigned)bestv : 0xFFFFFFFFu;
      vi = __reduce_min_sync(0xFFFFFFFFu, vi);
    }
    unsigned am = 0xFFFFFFFFu;
    if (lane == 0 && vi < (unsigned)nvec) {
      const uint4 xv = __ldg(p + vi);
      am = vi * VE + (unsigned)vec_first_eq<BF16>(xv, m);
    }
    if (lane == 0) {
      RowOut ro{m, s, w, am, 1.0f};
      write_row(a, row, lab, ro);
    }
  }
}

// ---------------------------------------------------------------------------
// K1a (async): the same grouped reduction, but the next row is prefetched with
// per-lane cp.async (16 B, L2-only) into a per-warp shared-memory double
// buffer instead of a second register set.  Each lane copies exactly the
// vectors it will reduce, so its own cp.async.wait_group is the only
// synchronisation (no barrier, no cross-lane hand-off).  Freeing the 32
// prefetch registers lets three CTAs (24 warps) share an SM, and the register
// copy B -> A disappears.
// ---------------------------------------------------------------------------
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool pred) {
  asm volatile(
      "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %2, 0;\n\t"
      "@p cp.async.cg.shared.global [%0], [%1], 16;\n\t}"
      ::"r"(dst), "l"(src), "r"((int)pred) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <int NV, int G, bool FULL>
__device__ __forceinline__ void group_prefetch_row(uint32_t sdst, const uint4* p, int gl, int nvec) {
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = k * G + gl;
    cp_async16(sdst + (uint32_t)(k * G * 16), p + vi, (FULL && k < NV - 1) || vi < nvec);
  }
}

template <bool BF16, int NV, int G, bool FULL>
__device__ __forceinline__ void group_lds_row(uint4 (&v)[NV], uint32_t ssrc, int gl, int nvec) {
  const uint32_t f = BF16 ? kBf16NegInf2 : kF32NegInf;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    const int vi = k * G + gl;
    uint4 r = make_uint4(f, f, f, f);
    if ((FULL && k < NV - 1) || vi < nvec)
      asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];"
                   : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "r"(ssrc + (uint32_t)(k * G * 16)));
    v[k] = r;
  }
}

// ---- fused threshold test + stable compaction (K1+K3, FuseArgs) ------------
// One cooperative launch (all CTAs co-resident).  Row groups are cut into at
// most kFuseTiles tiles of 2^s consecutive groups.  While streaming its rows a
// warp adds each group's deferred count to the group's tile counter (one
// relaxed reduction; no fence).  After the last row, ONE grid barrier; then
// every CTA scans the tile counters into exclusive deferred prefixes (shared
// memory, the same in every CTA) and each warp writes the accepted / deferred
// lists of its tiles in row order, reading the rows' confidences and
// argmaxes that the barrier made visible.  The counters alternate between two
// banks by launch (the launch epoch's parity): a launch zeroes the bank the
// next one uses.
struct FuseTiles {
  unsigned* epoch;
  unsigned* acc;          // [2][kFuseTiles]
};
__device__ __forceinline__ FuseTiles fuse_tiles(void* w) {
  char* b = reinterpret_cast<char*>(w);
  return {reinterpret_cast<unsigned*>(b), reinterpret_cast<unsigned*>(b + 32)};
}
// Tiles of 2^s row groups (RPW rows each), s the least with <= kFuseTiles tiles.
__device__ __forceinline__ int fuse_tshift(int64_t rows, int RPW) {
  const int64_t ng = (rows + RPW - 1) / RPW;
  int sh = 0;
  while (((ng + (int64_t(1) << sh) - 1) >> sh) > kFuseTiles) ++sh;
  return sh;
}

// Tile j of R rows, its exclusive deferred prefix `excl` known: D3 per row
// (accept iff c >= t; NaN defers; the last stage accepts all), the accepted
// list and the deferred list (the next stage's batch) in row order.
__device__ __noinline__ void fuse_scatter_tile(const ConfArgs& a, int64_t j, int64_t R, int64_t rows,
                                               long long excl, float thr) {
  const int lane = threadIdx.x & 31;
  const FuseArgs& z = a.fz;
  const int64_t base = j * R;
  const int tn = (int)(R < rows - base ? R : rows - base);
  const int64_t acc_base = base - excl;            // accepted rows before this tile
  const unsigned lt = lanemask_lt();
  int dsum = 0;                                    // deferred rows of the tile so far
  for (int p0 = 0; p0 < tn; p0 += 128) {
    float cv[4];
    int64_t idv[4];
    int32_t pv[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * 32 + lane;
      const int64_t i = base + p;
      const bool in = p < tn;
      cv[u] = in ? __ldcg(a.conf + i) : 0.f;
      idv[u] = (in && z.ids) ? __ldg(z.ids + i) : i;
      pv[u] = (in && z.acc_pred) ? __ldcg(a.argmax + i) : 0;
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int p = p0 + u * 32 + lane;
      const bool in = p < tn;
      const bool d = in && !(z.is_last || cv[u] >= thr);
      const unsigned bd = __ballot_sync(0xFFFFFFFFu, d);
      const int r = __popc(bd & lt);
      if (d) {
        const int64_t pos = excl + dsum + r;
        if (z.def_ids) z.def_ids[pos] = idv[u];
        if (z.def_pos) z.def_pos[pos] = base + p;
      } else if (in) {
        const int64_t pos = acc_base + p - (dsum + r);
        if (z.acc_ids) z.acc_ids[pos] = idv[u];
        if (z.acc_conf) z.acc_conf[pos] = cv[u];
        if (z.acc_pred) z.acc_pred[pos] = pv[u];
      }
      dsum += __popc(bd);
    }
  }
}

// After the grid barrier: the prefixes (every CTA), the lists (warp per tile),
// the counts and the epoch (CTA 0).  `spre`: >= kFuseTiles + 32 words of
// shared memory.
__device__ __noinline__ void fuse_finish(const ConfArgs& a, int64_t rows, int RPW, unsigned epoch,
                                         float thr, unsigned* spre) {
  const FuseTiles t = fuse_tiles(a.fz.tiles);
  const unsigned* acc = t.acc + (epoch & 1u) * kFuseTiles;
  const int tsh = fuse_tshift(rows, RPW);
  const int64_t R = (int64_t(1) << tsh) * RPW;
  const int NT = (int)((rows + R - 1) / R);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5, nthr = blockDim.x;
  constexpr int PER = kFuseTiles / 256;            // tiles per thread (256-thread CTAs)
  unsigned v[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    const int j = tid * PER + q;
    v[q] = j < NT ? __ldcg(acc + j) : 0u;
    sum += v[q];
  }
  // block exclusive scan of the per-thread sums (warp scans + warp totals)
  unsigned inc = sum;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned y = __shfl_up_sync(0xFFFFFFFFu, inc, o);
    if (lane >= o) inc += y;
  }
  unsigned* wtot = spre + kFuseTiles;
  if (lane == 31) wtot[warp] = inc;
  __syncthreads();
  unsigned wbase = 0;
  for (int w = 0; w < warp; ++w) wbase += wtot[w];
  unsigned run = wbase + inc - sum;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    spre[tid * PER + q] = run;
    run += v[q];
  }
  __syncthreads();
  const int64_t nwarps = ((int64_t)gridDim.x * nthr) >> 5;
  const int64_t gw = ((int64_t)blockIdx.x * nthr + tid) >> 5;
  for (int64_t j = gw; j < NT; j += nwarps) fuse_scatter_tile(a, j, R, rows, (long long)spre[j], thr);
  if (blockIdx.x == 0 && tid == 0) {
    unsigned total = 0;
    for (int w = 0; w < nthr / 32; ++w) total += wtot[w];
    a.fz.counts[0] = rows - (long long)total;
    a.fz.counts[1] = (long long)total;
    *(volatile unsigned*)t.epoch = epoch + 1u;     // every CTA read it before the barrier
  }
}

constexpr int kAsyncThreads = 256;
template <int NV, int G>
constexpr int async_smem_bytes() { return (kAsyncThreads / 32) * 2 * (32 / G) * G * NV * 16; }

// RIDX: the launch reads rows through row_index (gathered batch); false for
// dense batches -- the row-index lookups and checks compile away.
// FUSE: the threshold test + stable compaction of hs_cascade_step in the row
// epilogue (a.fz; requires DYN and no late wait).
template <bool BF16, bool ENTROPY, int NV, int G, bool FULL, bool DYN, bool RIDX, bool FUSE>
__global__ void __launch_bounds__(kAsyncThreads, 3) conf_async_kernel(const __grid_constant__ ConfArgs a) {
  static_assert(!(FUSE && DYN), "the fused compaction uses the static row assignment");
  // EARLY: static rows of a dense batch -- the warp's first row is prefetched
  // before waiting for the previous kernel (logits are never written by a libhs
  // kernel; only the live count is, and it is read after the wait), so the
  // first load's latency overlaps that kernel's drain
#ifdef HS_AB_NO_EARLY
  constexpr bool EARLY = false;
#else
  constexpr bool EARLY = !DYN && !RIDX;
#endif
  const bool early = EARLY && (a.rows_cap_valid || !a.d_n);
  if (a.late_wait || early) pdl_trigger(); else pdl_start();
  if (!a.late_wait && !early) write_last_counts(a);
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int RPW = 32 / G;
  constexpr uint32_t ROWB = G * NV * 16;              // one group's row slot
  constexpr uint32_t STAGEB = RPW * ROWB;             // one warp's stage
  const int lane = threadIdx.x & 31, gl = lane % G, grp = lane / G, warp = threadIdx.x >> 5;
  const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const int nvec = a.nvec;
  constexpr bool dyn = DYN;   // a.ticket != NULL
  // row-index reads are speculative within the capacity (capacity-sized
  // buffers), so they overlap the read of the device count *d_n
  const int64_t cap = a.n * a.L * (int64_t)a.nbatch;
  // row group g = rows g*RPW .. g*RPW + RPW-1: static (warp w takes w, w + nwarps,
  // ...) or claimed from the ticket, so CTAs that start late (SMs still busy with
  // the previous kernel) just take fewer groups
  // dynamic claims come in chunks of kChunk groups per warp (one atomic per
  // kChunk * RPW rows keeps the single ticket word off the critical path)
  // The next chunk is claimed when the current chunk's last group is handed
  // out and taken when that group has been reduced: the ticket atomic's
  // latency hides behind a row group, and a warp holds at most one group
  // beyond its current chunk (tail balance).
  // chunks of 8 row groups (A/B: chunks of 1-4 groups for small batches are
  // slower -- the single ticket word's atomics serialise)
  constexpr int kShift = 3;
  constexpr int kChunk = 1 << kShift;
  int64_t cnext = 0, cend = 0;
  unsigned cpre = 0;                                  // lane 0: the chunk claimed ahead
  auto claim = [&]() {
    if (lane == 0) cpre = atomicAdd(a.ticket, (unsigned)kChunk);
  };
  // fused: warps take blocks of 2^bsh consecutive row groups, strided (one
  // tile-counter reduction per block; small batches use smaller blocks)
  int bsh = 0;
  if constexpr (FUSE) {
    const int64_t lr = live_rows(a);
    const int64_t per = ((lr + RPW - 1) / RPW) / (4 * nwarps);
    bsh = per >= 8 ? 3 : per >= 4 ? 2 : per >= 2 ? 1 : 0;
    const int ts = fuse_tshift(lr, RPW);    // a block never straddles two tiles
    if (bsh > ts) bsh = ts;
#ifndef HS_FZ_BLOCKS
    bsh = 0;                                // A/B: blocks of consecutive groups were slower
#endif
  }
  auto next_group = [&](int64_t g) -> int64_t {
    if (!dyn) {
      if constexpr (FUSE) {
        const int64_t B = int64_t(1) << bsh;
        return ((g + 1) & (B - 1)) ? g + 1 : g + 1 + (nwarps - 1) * B;
      }
      return g + nwarps;
    }
    if (cnext == cend) {
      cnext = (int64_t)__shfl_sync(0xFFFFFFFFu, cpre, 0);
      cend = cnext + kChunk;
    }
    if (cnext == cend - 1) claim();
    return cnext++;
  };
  if (dyn) claim();
  const int64_t g0 = dyn ? next_group(0) : (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5) << bsh;
  const int64_t fA = fetch_index_t<RIDX>(a, g0 * RPW + grp < cap ? g0 * RPW + grp : 0);
  // lane gl's vector k of stage st sits at base + st*STAGEB + grp*ROWB + k*G*16 + gl*16:
  // a quarter-warp reads 128 contiguous bytes (conflict-free LDS.128)
  const uint32_t sbase = smem_u32(smem) + (uint32_t)warp * 2u * STAGEB + (uint32_t)grp * ROWB +
                         (uint32_t)gl * 16u;
  BatchCur cur = cur_init(a);
  const uint4* pA = nullptr;
  float cA = 0.f;
  int32_t labA = 0;
  auto locate_A = [&](bool actA) {
    const RowSrc r = locate_cur<RIDX>(a, cur, actA ? g0 * RPW + grp : 0,
                                      actA ? fA : fetch_index_t<RIDX>(a, 0));
    pA = reinterpret_cast<const uint4*>(r.base + r.src * a.row_bytes);
    cA = r.c;
    labA = fetch_label(a, r);
  };
  if constexpr (EARLY) {
    if (early && !a.late_wait) {
      if (g0 * RPW < cap) {                          // within the capacity: valid memory
        locate_A(g0 * RPW + grp < cap);
        group_prefetch_row<NV, G, FULL>(sbase, pA, gl, nvec);
      }
      cp_async_commit();
      pdl_wait();
      write_last_counts(a);
    }
  }
  const int64_t rows = live_rows(a);
  // fused compaction: tiles of 2^tsh row groups, counters in bank epoch & 1
  float thr = 0.f;
  int tsh = 0;
  unsigned epoch = 0, cdef = 0;
  unsigned* tacc = nullptr;
  if constexpr (FUSE) {
    thr = a.fz.d_threshold ? *a.fz.d_threshold : a.fz.threshold;
    tsh = fuse_tshift(rows, RPW);
    const FuseTiles t = fuse_tiles(a.fz.tiles);
    epoch = *(volatile unsigned*)t.epoch;
    tacc = t.acc + (epoch & 1u) * kFuseTiles;
    if (blockIdx.x == 0)                       // the next launch's bank
      for (int j = threadIdx.x; j < kFuseTiles; j += blockDim.x) t.acc[((epoch + 1u) & 1u) * kFuseTiles + j] = 0u;
  }
  if (g0 * RPW < rows) {
    // row A (being reduced) and row B (in flight) of this group: row pointer,
    // temperature factor, label; row C's gathered index is fetched one pass ahead
    int64_t rowA = g0 * RPW + grp;
    bool actA = rowA < rows;
    if (!(early && !a.late_wait)) {
      locate_A(actA);
      group_prefetch_row<NV, G, FULL>(sbase, pA, gl, nvec);
      cp_async_commit();
    } else if (!actA) {
      locate_A(false);                 // the early prefetch assumed a live row: re-aim
    }
    int64_t gA = g0;
    int64_t gB = next_group(g0);
    int64_t fB = fetch_index_t<RIDX>(a, gB * RPW + grp < cap ? gB * RPW + grp : 0);
    uint4 A[NV];
    for (int it = 0;; ++it) {
      const int64_t rowB = gB * RPW + grp;
      const bool anyB = gB * RPW < rows;      // warp-uniform
      const bool actB = rowB < rows;
      int64_t gC = 0, fC = 0;
      const uint4* pB = pA;
      float cB = cA;
      int32_t labB = 0;
      if (anyB) {
        const RowSrc r = locate_cur<RIDX>(a, cur, actB ? rowB : 0, actB ? fB : fetch_index_t<RIDX>(a, 0));
        pB = reinterpret_cast<const uint4*>(r.base + r.src * a.row_bytes);
        cB = r.c;
        group_prefetch_row<NV, G, FULL>(sbase + (uint32_t)((it + 1) & 1) * STAGEB, pB, gl, nvec);
        labB = fetch_label(a, r);
        gC = next_group(gB);
        const int64_t rowC = gC * RPW + grp;
        fC = fetch_index_t<RIDX>(a, rowC < cap ? rowC : 0);
      }
      cp_async_commit();
      cp_async_wait<1>();        // this lane's copies of row A have landed
      group_lds_row<BF16, NV, G, FULL>(A, sbase + (uint32_t)(it & 1) * STAGEB, gl, nvec);
      if (a.tail) group_mask_tail<BF16, NV, G>(A, gl, nvec, a.tail);
      const float crA = group_reduce_row<BF16, ENTROPY, NV, G>(a, A, actA, rowA, gl, cA, pA, labA);
      if constexpr (FUSE) {
        // D3 per row (accept iff c >= t, NaN defers; the last stage accepts
        // all): the group's deferred rows go to its tile's counter
        cdef += (unsigned)__popc(__ballot_sync(0xFFFFFFFFu, actA && gl == 0 && !(a.fz.is_last || crA >= thr)));
        if ((((gA + 1) >> bsh) << bsh) == gA + 1 || !anyB) {     // end of the warp's block
          if (lane == 0 && cdef) atomicAdd(tacc + (gA >> tsh), cdef);
          cdef = 0;
        }
      }
      if (!anyB) break;
      gA = gB;
      rowA = rowB;
      actA = actB;
      pA = pB;
      cA = cB;
      labA = labB;
      gB = gC;
      fB = fC;
    }
    cp_async_wait<0>();
  }
  if constexpr (EARLY) cp_async_wait<0>();     // an early prefetch of a row beyond the live count
  if constexpr (FUSE) {
#ifndef HS_EXP_FZ_NOSYNC
    cooperative_groups::this_grid().sync();    // every row's confidence, argmax and count
#ifndef HS_EXP_FZ_NOFINISH
    fuse_finish(a, rows, RPW, epoch, thr, reinterpret_cast<unsigned*>(smem));
#endif
#endif
  }
  if (dyn) {
    // the claim issued ahead must have landed before the last CTA re-arms the
    // ticket: consume its result (the store below never executes -- ticket
    // values are multiples of kChunk -- but keeps the wait from being elided)
    cpre = __shfl_sync(0xFFFFFFFFu, cpre, 0);
    if (cpre == 0xFFFFFFFFu) a.ticket[2] = 0u;
    __syncthreads();                 // every warp of this CTA is done claiming
    if (threadIdx.x == 0) {
      const unsigned done = atomicAdd(a.ticket + 1, 1u);
      if (done == gridDim.x - 1) {   // last CTA: rearm for the next launch
        a.ticket[0] = 0u;
        a.ticket[1] = 0u;
      }
    }
  }
  if (a.late_wait) {
    pdl_wait();                      // completes only after the previous kernel
    write_last_counts(a);
  }
}

// ---------------------------------------------------------------------------
// K1a': the same grouped reduction, rows staged into shared memory by the TMA
// engine (cp.async.bulk + mbarrier ring).  Warp 0 is the producer: lane 0 arms
// the stage's "full" barrier with the tile's byte count, the lanes issue one
// bulk copy per row (gathered rows) or one per tile (dense rows), with an L2
// evict-first policy.  Warps 1..NCW consume 32/G rows each per stage (LDS.128,
// conflict-free), reduce them in registers and release the stage through the
// "empty" barrier.  S stages keep S*NCW*32/G rows in flight per SM.
// ---------------------------------------------------------------------------
template <int S>
struct TmaRing {
  uint64_t full[S];
  uint64_t empty[S];
};

template <bool BF16, bool ENTROPY, int NV, int G, int NCW, int S, bool L1>
__global__ void __launch_bounds__(32 * (NCW + 1), 1) conf_tma_kernel(const ConfArgs a, int dense) {
  pdl_start();
  write_last_counts(a);
  extern __shared__ __align__(128) unsigned char smem[];
  constexpr int RPW = 32 / G;
  constexpr int RPS = NCW * RPW;          // rows per stage
  TmaRing<S>* ring = reinterpret_cast<TmaRing<S>*>(smem);
  unsigned char* stage_base = smem + 128 * ((sizeof(TmaRing<S>) + 127) / 128);
  const int nvec = a.nvec;
  const uint32_t row_sm = (uint32_t)nvec * 16u;
  const uint32_t stage_bytes = row_sm * RPS;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t rows = live_rows(a);
  const int64_t ntiles = (rows + RPS - 1) / RPS;

  if (threadIdx.x == 0) {
    for (int i = 0; i < S; ++i) {
      mbar_init(&ring->full[i], 1);
      mbar_init(&ring->empty[i], NCW);
    }
    fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer ----------------
    const uint64_t pol = policy_evict_first();
    const char* base = (const char*)a.logits;
    int it = 0;
    for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
      const int st = it % S;
      const uint32_t ph = (uint32_t)(it / S) & 1u;
      const int64_t r0 = t * RPS;
      const int nr = (int)min((int64_t)RPS, rows - r0);
      if (lane == 0) {
        mbar_wait(&ring->empty[st], ph ^ 1u);
        mbar_arrive_expect_tx(&ring->full[st], row_sm * (uint32_t)nr);
      }
      __syncwarp();
      unsigned char* dst = stage_base + (size_t)st * stage_bytes;
      if (dense && !a.row_index) {
        if (lane == 0)
          bulk_g2s(dst, base + r0 * a.row_bytes, row_sm * (uint32_t)nr, &ring->full[st], pol);
      } else {
        for (int j = lane; j < nr; j += 32)
          bulk_g2s(dst + (size_t)j * row_sm, base + src_row<L1>(a, r0 + j) * a.row_bytes, row_sm,
                   &ring->full[st], pol);
      }
    }
    return;
  }
  // ---------------- consumers ----------------
  const int cw = warp - 1, gl = lane % G, grp = lane / G;
  const uint32_t f = BF16 ? kBf16NegInf2 : kF32NegInf;
  int it = 0;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x, ++it) {
    const int st = it % S;
    const uint32_t ph = (uint32_t)(it / S) & 1u;
    const int slot = cw * RPW + grp;
    const int64_t row = t * RPS + slot;
    const bool act = row < rows;
    mbar_wait(&ring->full[st], ph);
    const unsigned char* srow = stage_base + (size_t)st * stage_bytes + (size_t)slot * row_sm;
    const int lim = act ? nvec : 0;
    uint4 v[NV];
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int vi = k * G + gl;
      v[k] = vi < lim ? lds128(srow + (size_t)vi * 16) : make_uint4(f, f, f, f);
    }
    if (a.tail) group_mask_tail<BF16, NV, G>(v, gl, nvec, a.tail);
    const int64_t src = act ? src_row<L1>(a, row) : 0;
    group_reduce_row<BF16, ENTROPY, NV, G>(a, v, act, row, gl, a.c,
                                           reinterpret_cast<const uint4*>((const char*)a.logits + src * a.row_bytes),
                                           a.labels ? __ldg(a.labels + src) : 0);
    // every lane has consumed its staged vectors (the row max read them all)
    __syncwarp();
    if (lane == 0) mbar_arrive(&ring->empty[st]);
  }
}

// ---------------------------------------------------------------------------
// K1b: one CTA per row (persistent over rows), per-thread online softmax over
// chunks of NV vectors per thread, block merge at the end of each row.  The
// CTA walks its (row, chunk) items in order and always has the next item's
// loads in flight while reducing the current one; chunks fully inside the row
// load unconditionally (no per-vector predicate/default moves).
// ---------------------------------------------------------------------------
template <bool BF16, int NV, int NT>
__device__ __forceinline__ void cta_load_chunk(uint4 (&v)[NV], const uint4* p, int base, int tid,
                                               int nvec, int tail, bool full) {
  const uint32_t f = BF16 ? kBf16NegInf2 : kF32NegInf;
  if (full) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] = ldg_stream(p + base + k * NT + tid);
  } else {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      const int vi = base + k * NT + tid;
      uint4 r = make_uint4(f, f, f, f);
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.lt.s32 p, %4, %5;\n\t"
          "@p ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%6];\n\t}"
          : "+r"(r.x), "+r"(r.y), "+r"(r.z), "+r"(r.w)
          : "r"(vi), "r"(nvec), "l"(p + vi));
      v[k] = r;
    }
    if (tail) {
#pragma unroll
      for (int k = 0; k < NV; ++k) {
        const bool q = (base + k * NT + tid) == nvec - 1;
        const uint4 m = masked<BF16>(v[k], tail);
        v[k] = make_uint4(q ? m.x : v[k].x, q ? m.y : v[k].y, q ? m.z : v[k].z, q ? m.w : v[k].w);
      }
    }
  }
}

template <bool BF16, bool ENTROPY, int NT, int NV>
__global__ void __launch_bounds__(NT) conf_cta_kernel(const ConfArgs a) {
  pdl_start();
  write_last_counts(a);
  constexpr int NW = NT / 32;
  constexpr int VE = BF16 ? 8 : 4;
  constexpr int CH = NT * NV;                  // vectors per chunk
  __shared__ float sh_m[NW], sh_s[NW], sh_w[NW];
  __shared__ unsigned sh_am[NW];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t rows = live_rows(a);
  const int nvec = a.nvec;
  const int nch = (nvec + CH - 1) / CH;
  if ((int64_t)blockIdx.x >= rows) return;
  // (row, chunk) items of this CTA in order; the next one is always in flight
  int64_t rowA = blockIdx.x;
  int chA = 0;
  RowSrc rsA = locate(a, rowA), rsB = rsA;
  const uint4* pA = reinterpret_cast<const uint4*>(rsA.base + rsA.src * a.row_bytes);
  const uint4* pB = pA;
  uint4 A[NV], B[NV];
  cta_load_chunk<BF16, NV, NT>(A, pA, 0, tid, nvec, a.tail, CH <= nvec);

  float m = -INFINITY;
  int mch = -1;                                // chunk where the running max was set
  f2_t s2 = f2(0.f, 0.f), w2 = f2(0.f, 0.f);
  while (true) {
    // ---- next item: same row, next chunk; or the next row of this CTA
    int64_t rowB = rowA;
    int chB = chA + 1;
    if (chB == nch) {
      chB = 0;
      rowB = rowA + gridDim.x;
    }
    const bool more = rowB < rows;
    if (more) {
      if (chB == 0) {
        rsB = locate(a, rowB);
        pB = reinterpret_cast<const uint4*>(rsB.base + rsB.src * a.row_bytes);
      }
      cta_load_chunk<BF16, NV, NT>(B, pB, chB * CH, tid, nvec, a.tail, (chB + 1) * CH <= nvec);
    }
    const float c = rsA.c;
    const f2_t c2 = f2(c, c);
    // ---- chunk max; a new running max rescales (s, w); argmax located at row end
    float cm = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) cm = fmax_nan(cm, vec_max<BF16>(A[k]));
    if (!(cm <= m)) {
      const float nm = fmax_nan(m, cm);
      if (m > -INFINITY) {
        const float d = (m - nm) * c;
        const float f = ex2(d);
        const f2_t f2v = f2(f, f);
        if (ENTROPY) w2 = f2mul(f2v, f2fma(f2(d, d), s2, w2));
        s2 = f2mul(f2v, s2);
      }
      m = nm;
      mch = chA;
    }
    if (m > -INFINITY) {
      const f2_t m2 = f2(m, m);
      const uint32_t cw = ENTROPY && BF16 ? entropy_clamp_word(m, c) : 0u;
#pragma unroll
      for (int k = 0; k < NV; ++k) vec_accum<BF16, ENTROPY>(A[k], m2, c2, cw, s2, w2);
    }
    if (chA == nch - 1) {
      // ---- block merge: max, rescale to it, fixed-order sums, min index among maxima
      float M = m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmax_nan(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
      if (lane == 0) sh_m[wid] = M;
      __syncthreads();
      M = sh_m[0];
#pragma unroll
      for (int i = 1; i < NW; ++i) M = fmax_nan(M, sh_m[i]);
      float sv = 0.f, wv = 0.f;
      if (m > -INFINITY) {
        const float d = (m - M) * c;
        const float f = ex2(d);
        const float ls = f2lo(s2) + f2hi(s2);
        sv = f * ls;
        if (ENTROPY && f > 0.f) wv = f * ((f2lo(w2) + f2hi(w2)) + d * ls);
      }
      sv = warp_sum(sv);
      if (ENTROPY) wv = warp_sum(wv);
      // argmax: a thread holding M re-reads the chunk where it first saw its
      // max (rare, L2-hot) and finds the lowest index equal to M
      unsigned mine = 0xFFFFFFFFu;
      if (m == M && mch >= 0) {
        uint4 R[NV];
        const uint4* pr = reinterpret_cast<const uint4*>(rsA.base + rsA.src * a.row_bytes);
        cta_load_chunk<BF16, NV, NT>(R, pr, mch * CH, tid, nvec, a.tail, (mch + 1) * CH <= nvec);
#pragma unroll
        for (int k = NV - 1; k >= 0; --k) {
          const int e = vec_first_eq<BF16>(R[k], M);
          if (e < VE) mine = (unsigned)((mch * CH + k * NT + tid) * VE + e);
        }
      }
      const unsigned wam = __reduce_min_sync(0xFFFFFFFFu, mine);
      if (lane == 0) {
        sh_s[wid] = sv;
        sh_w[wid] = wv;
        sh_am[wid] = wam;
      }
      __syncthreads();
      if (tid == 0) {
        float S = 0.f, W = 0.f;
        unsigned AM = 0xFFFFFFFFu;
#pragma unroll
        for (int i = 0; i < NW; ++i) {
          S += sh_s[i];
          W += sh_w[i];
          AM = min(AM, sh_am[i]);
        }
        RowOut r{M, S, W, AM, 1.0f};
        write_row(a, rowA, a.labels ? __ldg(a.labels + rsA.src) : 0, r);
      }
      __syncthreads();
      m = -INFINITY;
      mch = -1;
      s2 = f2(0.f, 0.f);
      w2 = f2(0.f, 0.f);
    }
    if (!more) break;
#pragma unroll
    for (int k = 0; k < NV; ++k) A[k] = B[k];
    rowA = rowB;
    chA = chB;
    rsA = rsB;
  }
}

// ---------------------------------------------------------------------------
// K1d: one WARP per vocabulary-sized row (persistent over rows), the same
// per-lane online (max, sum, weighted sum) over chunks of 32 x NV vectors as
// K1b, the next (row, chunk) item in flight; the row merge is a warp merge
// (shuffles), so no CTA barrier ever stalls the other rows' streams (K1b's top
// stall on T5 rows: barrier 1.5 warps per issue).
// ---------------------------------------------------------------------------
template <bool BF16, bool ENTROPY, int NV>
__global__ void __launch_bounds__(256, 2) conf_stream_kernel(const ConfArgs a) {
  pdl_start();
  write_last_counts(a);
  constexpr int VE = BF16 ? 8 : 4;
  constexpr int CH = 32 * NV;                  // vectors per chunk
  const int lane = threadIdx.x & 31;
  const int64_t rows = live_rows(a);
  const int nvec = a.nvec;
  const int nch = (nvec + CH - 1) / CH;
  const int64_t nwarps = (int64_t)gridDim.x * (blockDim.x >> 5);
  int64_t rowA = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (rowA >= rows) return;
  int chA = 0;
  RowSrc rsA = locate(a, rowA), rsB = rsA;
  const uint4* pB = reinterpret_cast<const uint4*>(rsA.base + rsA.src * a.row_bytes);
  uint4 A[NV], B[NV];
  cta_load_chunk<BF16, NV, 32>(A, pB, 0, lane, nvec, a.tail, CH <= nvec);
  int32_t labA = (a.labels && lane == 0) ? __ldg(a.labels + rsA.src) : 0, labB = 0;

  float m = -INFINITY;
  int mch = -1;                                // chunk where the lane's running max was set
  f2_t s2 = f2(0.f, 0.f), w2 = f2(0.f, 0.f);
  while (true) {
    int64_t rowB = rowA;
    int chB = chA + 1;
    if (chB == nch) {
      chB = 0;
      rowB = rowA + nwarps;
    }
    const bool more = rowB < rows;
    if (more) {
      if (chB == 0) {
        rsB = locate(a, rowB);
        pB = reinterpret_cast<const uint4*>(rsB.base + rsB.src * a.row_bytes);
        if (a.labels && lane == 0) labB = __ldg(a.labels + rsB.src);
      }
      cta_load_chunk<BF16, NV, 32>(B, pB, chB * CH, lane, nvec, a.tail, (chB + 1) * CH <= nvec);
    }
    const float c = rsA.c;
    const f2_t c2 = f2(c, c);
    float cm = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) cm = fmax_nan(cm, vec_max<BF16>(A[k]));
    if (!(cm <= m)) {
      const float nm = fmax_nan(m, cm);
      if (m > -INFINITY) {
        const float d = (m - nm) * c;
        const float f = ex2(d);
        const f2_t f2v = f2(f, f);
        if (ENTROPY) w2 = f2mul(f2v, f2fma(f2(d, d), s2, w2));
        s2 = f2mul(f2v, s2);
      }
      m = nm;
      mch = chA;
    }
    if (m > -INFINITY) {
      // the chunk's terms are summed apart and then added to the row's running
      // sums: each lane adds ~4,000 terms on a Llama row, a single running fp32
      // sum would exceed the 1e-5 tolerance
      const f2_t m2 = f2(m, m);
      const uint32_t cw = ENTROPY && BF16 ? entropy_clamp_word(m, c) : 0u;
      f2_t cs = f2(0.f, 0.f), cwv = f2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < NV; ++k) vec_accum<BF16, ENTROPY>(A[k], m2, c2, cw, cs, cwv);
      s2 = f2add(s2, cs);
      if (ENTROPY) w2 = f2add(w2, cwv);
    }
    if (chA == nch - 1) {
      // ---- warp merge: max, rescale to it, fixed-order sums, min index among maxima
      float M = m;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) M = fmax_nan(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
      float sv = 0.f, wv = 0.f;
      if (m > -INFINITY) {
        const float d = (m - M) * c;
        const float f = ex2(d);
        const float ls = f2lo(s2) + f2hi(s2);
        sv = f * ls;
        if (ENTROPY && f > 0.f) wv = f * ((f2lo(w2) + f2hi(w2)) + d * ls);
      }
      sv = warp_sum(sv);
      if (ENTROPY) wv = warp_sum(wv);
      unsigned mine = 0xFFFFFFFFu;
      if (m == M && mch >= 0) {      // re-read the lane's vectors of the chunk that set its max (L2-hot)
        uint4 R[NV];
        const uint4* pr = reinterpret_cast<const uint4*>(rsA.base + rsA.src * a.row_bytes);
        cta_load_chunk<BF16, NV, 32>(R, pr, mch * CH, lane, nvec, a.tail, (mch + 1) * CH <= nvec);
#pragma unroll
        for (int k = NV - 1; k >= 0; --k) {
          const int e = vec_first_eq<BF16>(R[k], M);
          if (e < VE) mine = (unsigned)((mch * CH + k * 32 + lane) * VE + e);
        }
      }
      const unsigned am = __reduce_min_sync(0xFFFFFFFFu, mine);
      if (lane == 0) {
        RowOut r{M, sv, wv, am, 1.0f};
        write_row(a, rowA, labA, r);
      }
      m = -INFINITY;
      mch = -1;
      s2 = f2(0.f, 0.f);
      w2 = f2(0.f, 0.f);
      labA = labB;
    }
    if (!more) break;
#pragma unroll
    for (int k = 0; k < NV; ++k) A[k] = B[k];
    rowA = rowB;
    chA = chB;
    rsA = rsB;
  }
}

// ---------------------------------------------------------------------------
// K1e: split rows for small batches of long rows (routing latency, Fig. 8
// P:1039-1040).  Row r is cut into S contiguous segments of whole chunks, one
// warp each (K1d's per-lane online reduction); each warp publishes its
// segment's (max, sum, weighted sum, first argmax) and the LAST warp of the row
// to arrive (per-row arrival counter) merges the S partials in segment order
// (fixed tree: deterministic) and writes the row; it re-arms the counter.
// ---------------------------------------------------------------------------
struct SplitPart {
  float m, s, w;
  uint32_t am;
};

// (m, s, w) relative to m (base-2 exponents scaled by c), folded into the running
// (M, S, W, AM) -- the same rescale as K1b/K1d's row merge
__device__ __forceinline__ void fold_part(float& M, float& S, float& W, uint32_t& AM, const SplitPart& q,
                                          float c, bool ent) {
  const float nm = fmax_nan(M, q.m);
  float s0 = 0.f, w0 = 0.f, s1 = 0.f, w1 = 0.f;
  if (M > -INFINITY && nm == nm) {
    const float d = (M - nm) * c, f = ex2(d);
    s0 = f * S;
    if (ent && f > 0.f) w0 = f * (W + d * S);
  }
  if (q.m > -INFINITY && nm == nm) {
    const float d = (q.m - nm) * c, f = ex2(d);
    s1 = f * q.s;
    if (ent && f > 0.f) w1 = f * (q.w + d * q.s);
  }
  AM = (M == nm ? AM : 0xFFFFFFFFu);
  if (q.m == nm) AM = min(AM, q.am);
  M = nm;
  S = s0 + s1;
  W = w0 + w1;
}

template <bool BF16, bool ENTROPY, int NV>
__global__ void __launch_bounds__(256) conf_split_kernel(const ConfArgs a, int nseg, int segch,
                                                         SplitPart* parts, unsigned* arrive) {
  pdl_start();
  write_last_counts(a);
  constexpr int VE = BF16 ? 8 : 4;
  constexpr int CH = 32 * NV;
  const int lane = threadIdx.x & 31;
  const int64_t gw = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int64_t row = gw / nseg;
  const int seg = (int)(gw - row * nseg);
  if (row >= live_rows(a)) return;
  const int nvec = a.nvec;
  const int nch = (nvec + CH - 1) / CH;
  const int c0 = seg * segch, c1 = min(nch, c0 + segch);
  const RowSrc rs = locate(a, row);
  const uint4* p = reinterpret_cast<const uint4*>(rs.base + rs.src * a.row_bytes);
  const float c = rs.c;
  const f2_t c2 = f2(c, c);
  float m = -INFINITY;
  int mch = -1;
  f2_t s2 = f2(0.f, 0.f), w2 = f2(0.f, 0.f);
  uint4 A[NV], B[NV];
  cta_load_chunk<BF16, NV, 32>(A, p, c0 * CH, lane, nvec, a.tail, (c0 + 1) * CH <= nvec);
  for (int ch = c0; ch < c1; ++ch) {
    const bool more = ch + 1 < c1;
    if (more) cta_load_chunk<BF16, NV, 32>(B, p, (ch + 1) * CH, lane, nvec, a.tail, (ch + 2) * CH <= nvec);
    float cm = -INFINITY;
#pragma unroll
    for (int k = 0; k < NV; ++k) cm = fmax_nan(cm, vec_max<BF16>(A[k]));
    if (!(cm <= m)) {
      const float nm = fmax_nan(m, cm);
      if (m > -INFINITY) {
        const float d = (m - nm) * c;
        const float f = ex2(d);
        const f2_t f2v = f2(f, f);
        if (ENTROPY) w2 = f2mul(f2v, f2fma(f2(d, d), s2, w2));
        s2 = f2mul(f2v, s2);
      }
      m = nm;
      mch = ch;
    }
    if (m > -INFINITY) {
      const f2_t m2 = f2(m, m);
      const uint32_t cw = ENTROPY && BF16 ? entropy_clamp_word(m, c) : 0u;
      f2_t cs = f2(0.f, 0.f), cwv = f2(0.f, 0.f);
#pragma unroll
      for (int k = 0; k < NV; ++k) vec_accum<BF16, ENTROPY>(A[k], m2, c2, cw, cs, cwv);
      s2 = f2add(s2, cs);
      if (ENTROPY) w2 = f2add(w2, cwv);
    }
    if (more) {
#pragma unroll
      for (int k = 0; k < NV; ++k) A[k] = B[k];
    }
  }
  // ---- the segment's partial: warp merge (as K1d's row merge)
  float M = m;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) M = fmax_nan(M, __shfl_xor_sync(0xFFFFFFFFu, M, o));
  float sv = 0.f, wv = 0.f;
  if (m > -INFINITY) {
    const float d = (m - M) * c;
    const float f = ex2(d);
    const float ls = f2lo(s2) + f2hi(s2);
    sv = f * ls;
    if (ENTROPY && f > 0.f) wv = f * ((f2lo(w2) + f2hi(w2)) + d * ls);
  }
  sv = warp_sum(sv);
  if (ENTROPY) wv = warp_sum(wv);
  unsigned mine = 0xFFFFFFFFu;
  if (m == M && mch >= 0) {
    uint4 R[NV];
    cta_load_chunk<BF16, NV, 32>(R, p, mch * CH, lane, nvec, a.tail, (mch + 1) * CH <= nvec);
#pragma unroll
    for (int k = NV - 1; k >= 0; --k) {
      const int e = vec_first_eq<BF16>(R[k], M);
      if (e < VE) mine = (unsigned)((mch * CH + k * 32 + lane) * VE + e);
    }
  }
  const unsigned am = __reduce_min_sync(0xFFFFFFFFu, mine);
  unsigned last = 0;
  if (lane == 0) {
    parts[row * nseg + seg] = SplitPart{M, sv, wv, am};
    __threadfence();
    last = atomicAdd(arrive + row, 1u) == (unsigned)(nseg - 1);
  }
  if (!__shfl_sync(0xFFFFFFFFu, last, 0)) return;
  // ---- last arrival: merge the row's partials in segment order
  __threadfence();
  float RM = -INFINITY, RS = 0.f, RW = 0.f;
  uint32_t RA = 0xFFFFFFFFu;
  for (int j = lane; j < nseg; j += 32) {
    const float4 q4 = __ldcg(reinterpret_cast<const float4*>(parts + row * nseg + j));
    fold_part(RM, RS, RW, RA, SplitPart{q4.x, q4.y, q4.z, __float_as_uint(q4.w)}, c, ENTROPY);
  }
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {        // fixed tree over the lanes
    SplitPart q{__shfl_xor_sync(0xFFFFFFFFu, RM, o), __shfl_xor_sync(0xFFFFFFFFu, RS, o),
                __shfl_xor_sync(0xFFFFFFFFu, RW, o), __shfl_xor_sync(0xFFFFFFFFu, RA, o)};
    // both lanes of a pair must combine in the same order to stay identical
    if (lane & o) {
      const SplitPart mineq{RM, RS, RW, RA};
      RM = q.m; RS = q.s; RW = q.w; RA = q.am;
      fold_part(RM, RS, RW, RA, mineq, c, ENTROPY);
    } else {
      fold_part(RM, RS, RW, RA, q, c, ENTROPY);
    }
  }
  if (lane == 0) {
    RowOut r{RM, RS, RW, RA, 1.0f};
    write_row(a, row, a.labels ? __ldg(a.labels + rs.src) : 0, r);
    arrive[row] = 0u;                        // re-armed for the next launch (stream order)
  }
}

// ---------------------------------------------------------------------------
// K2: token -> sequence reduce, fixed order (P:423 MIN; MEAN), all-L correctness.
// ---------------------------------------------------------------------------
__global__ void seq_reduce_kernel(const float* tok_conf, const uint8_t* tok_ok, int64_t n,
                                  const int64_t* d_n, int L, int reduce, float* conf,
                                  uint8_t* correct) {
  pdl_start();
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

template <bool BF16, bool ENTROPY, int NV, int G, bool FULL>
int warp_occ() {
  static const int o = occupancy(conf_warp_kernel<BF16, ENTROPY, NV, G, FULL>, 256);
  return o;
}

template <bool BF16, bool ENTROPY, int NV, int G, bool FULL>
cudaError_t launch_warp_l(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_warp_kernel<BF16, ENTROPY, NV, G, FULL>;
  const int occ = warp_occ<BF16, ENTROPY, NV, G, FULL>();
  constexpr int RPB = 8 * (32 / G);      // rows per 256-thread block per pass
  const int64_t want = (rows + RPB - 1) / RPB;
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  return launch_pdl(k, dim3(grid), dim3(256), 0, s, a);
}

template <bool BF16, bool ENTROPY, int NV, int G, bool FULL, bool DYN, bool RIDX, bool FUSE = false>
cudaError_t launch_async_d(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_async_kernel<BF16, ENTROPY, NV, G, FULL, DYN, RIDX, FUSE>;
  constexpr int smem = async_smem_bytes<NV, G>();
  static const int occ = [&] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, kAsyncThreads, smem);
    return b > 0 ? b : 1;
  }();
  constexpr int RPB = (kAsyncThreads / 32) * (32 / G);
  const int64_t want = (rows + RPB - 1) / RPB;
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  if constexpr (FUSE) {
    // cooperative (one grid barrier; every CTA resident) + programmatic
    // dependent launch; the grid never exceeds one wave
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(kAsyncThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = pdl_enabled() ? 2 : 1;
    const cudaError_t e = cudaLaunchKernelEx(&cfg, k, a);
    count_launch();
    return e != cudaSuccess ? e : cudaGetLastError();
  }
  return launch_pdl(k, dim3(grid), dim3(kAsyncThreads), smem, s, a);
}

template <bool BF16, bool ENTROPY, int NV, int G, bool FULL>
cudaError_t launch_async_l(const ConfArgs& a, int64_t rows, cudaStream_t s) {
#ifdef HS_AB_K1_RIDX_ALWAYS
  if (true)
#else
  if (a.row_index)
#endif
  {
    if (a.fz.on) return launch_async_d<BF16, ENTROPY, NV, G, FULL, false, true, true>(a, rows, s);
    return a.ticket ? launch_async_d<BF16, ENTROPY, NV, G, FULL, true, true>(a, rows, s)
                    : launch_async_d<BF16, ENTROPY, NV, G, FULL, false, true>(a, rows, s);
  }
  if (a.fz.on) return launch_async_d<BF16, ENTROPY, NV, G, FULL, false, false, true>(a, rows, s);
  return a.ticket ? launch_async_d<BF16, ENTROPY, NV, G, FULL, true, false>(a, rows, s)
                  : launch_async_d<BF16, ENTROPY, NV, G, FULL, false, false>(a, rows, s);
}

int conf_impl();

template <bool BF16, bool ENTROPY, int NV, int G>
cudaError_t launch_warp(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  if constexpr (NV <= 8) {   // the async variant holds one row set in registers (<= 80 regs)
    if (conf_impl() == 2)
      return (NV - 1) * G <= a.nvec ? launch_async_l<BF16, ENTROPY, NV, G, true>(a, rows, s)
                                    : launch_async_l<BF16, ENTROPY, NV, G, false>(a, rows, s);
  }
#ifdef HS_NO_FULL
  return launch_warp_l<BF16, ENTROPY, NV, G, false>(a, rows, s);
#endif
  return (NV - 1) * G <= a.nvec ? launch_warp_l<BF16, ENTROPY, NV, G, true>(a, rows, s)
                                : launch_warp_l<BF16, ENTROPY, NV, G, false>(a, rows, s);
}

template <bool BF16, bool ENTROPY, int NT>
cudaError_t launch_cta(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_cta_kernel<BF16, ENTROPY, NT, 8>;
  static const int occ = occupancy(k, NT);
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(rows < cap ? (rows > 0 ? rows : 1) : cap);
  return launch_pdl(k, dim3(grid), dim3(NT), 0, s, a);
}

template <bool BF16, bool ENTROPY>
cudaError_t launch_stream(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_stream_kernel<BF16, ENTROPY, 8>;
  static const int occ = occupancy(k, 256);
  const int64_t want = (rows + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  return launch_pdl(k, dim3(grid), dim3(256), 0, s, a);
}

// K1e when the batch is too small to fill the GPU with one warp per row
template <bool BF16, bool ENTROPY>
bool launch_split(const ConfArgs& a, int64_t rows, cudaStream_t s, cudaError_t* err) {
  constexpr int NV = 8, CH = 32 * NV;
  if (!a.split_ws || a.top_k || a.ticket || rows > kSplitMaxRows || rows < 1) return false;
  static const bool off = getenv("HS_NO_SPLIT") && getenv("HS_NO_SPLIT")[0] == '1';
  if (off) return false;
  const int nch = (a.nvec + CH - 1) / CH;
  const int64_t target = (int64_t)num_sms() * 16;          // K1d's resident warps
  // measured (tools/fig8_sweep.py): splitting pays when every row gets >= 4
  // segments and rows are >= 8 chunks (>= 32 KB); below that the extra merge
  // costs more than the parallelism gains
  if (rows * 4 > target || nch < 8) return false;
  int64_t want = (target + rows - 1) / rows;
  if (want > kSplitMaxSeg) want = kSplitMaxSeg;
  if (want > nch) want = nch;
  if (want < 2) return false;
  const int segch = (int)((nch + want - 1) / want);
  const int nseg = (nch + segch - 1) / segch;
  if (nseg < 2) return false;
  SplitPart* parts = reinterpret_cast<SplitPart*>(reinterpret_cast<char*>(a.split_ws) +
                                                  (size_t)kSplitMaxRows * sizeof(unsigned));
  unsigned* arrive = reinterpret_cast<unsigned*>(a.split_ws);
  const int64_t warps = rows * nseg;
  if (a.split_zero) {
    *err = cudaMemsetAsync(arrive, 0, (size_t)rows * sizeof(unsigned), s);
    if (*err != cudaSuccess) return true;
  }
  *err = launch_pdl(conf_split_kernel<BF16, ENTROPY, NV>, dim3((unsigned)((warps + 7) / 8)), dim3(256), 0,
                    s, a, nseg, segch, parts, arrive);
  return true;
}

template <bool BF16, bool ENTROPY, int NV, int G, int NCW, int S, bool L1>
cudaError_t launch_tma_l(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_tma_kernel<BF16, ENTROPY, NV, G, NCW, S, L1>;
  constexpr int RPS = NCW * (32 / G);
  const size_t ring = 128 * ((sizeof(TmaRing<S>) + 127) / 128);
  const size_t smem = ring + (size_t)S * RPS * (size_t)a.nvec * 16;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024);
    attr = true;
  }
  const int64_t tiles = (rows + RPS - 1) / RPS;
  const int64_t cap = num_sms();
  const int grid = (int)(tiles < cap ? (tiles > 0 ? tiles : 1) : cap);
  const int dense = (a.row_bytes == (int64_t)a.nvec * 16) ? 1 : 0;
  return launch_pdl(k, dim3(grid), dim3(32 * (NCW + 1)), smem, s, a, dense);
}

// default TMA ring shape: 8 consumer warps, 3 stages (<= 3 x 64 KB of rows)
template <bool BF16, bool ENTROPY, int NV, int G, int NCW = 8, int S = 3>
cudaError_t launch_tma(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  return a.L == 1 ? launch_tma_l<BF16, ENTROPY, NV, G, NCW, S, true>(a, rows, s)
                  : launch_tma_l<BF16, ENTROPY, NV, G, NCW, S, false>(a, rows, s);
}

// 2 = cp.async double buffer (default; A/B on two boxes: +2.6 % and +9.6 % K1
// bandwidth over 0), 0 = LDG register double buffer, 1 = TMA bulk ring
int conf_impl() {
  static const int v = [] {
    const char* e = getenv("HS_CONF_IMPL");
    if (e && strcmp(e, "tma") == 0) return 1;
    if (e && strcmp(e, "ldg") == 0) return 0;
    if (e && strcmp(e, "cta") == 0) return 3;     // vocabulary rows: K1b instead of K1d
    return 2;
  }();
  return v;
}

// Row shapes: G lanes per row, NV 16-byte vectors per lane (G * NV >= nvec).
template <bool BF16, bool ENTROPY>
cudaError_t dispatch(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  const int nvec = a.nvec;
  if (nvec <= 512 && conf_impl() == 1 && a.nbatch == 1) {
    if (nvec <= 4) return launch_tma<BF16, ENTROPY, 1, 4>(a, rows, s);
    if (nvec <= 16) return launch_tma<BF16, ENTROPY, 4, 4>(a, rows, s);
    if (nvec <= 64) return launch_tma<BF16, ENTROPY, 16, 4>(a, rows, s);
    if (nvec <= 128) return launch_tma<BF16, ENTROPY, 16, 8>(a, rows, s);
    if (nvec <= 256) return launch_tma<BF16, ENTROPY, 16, 16>(a, rows, s);
    return launch_tma<BF16, ENTROPY, 16, 32>(a, rows, s);
  }
  if (nvec <= 4) return launch_warp<BF16, ENTROPY, 1, 4>(a, rows, s);
  if (nvec <= 16) return launch_warp<BF16, ENTROPY, 4, 4>(a, rows, s);
  if (nvec <= 32) return launch_warp<BF16, ENTROPY, 8, 4>(a, rows, s);
  if (nvec <= 64) return launch_warp<BF16, ENTROPY, 8, 8>(a, rows, s);
#ifdef HS_AB_K1A_G32
  if (nvec <= 128) return launch_warp<BF16, ENTROPY, 4, 32>(a, rows, s);   // A/B: one row per warp
#endif
  if (nvec <= 128) return launch_warp<BF16, ENTROPY, 8, 16>(a, rows, s);
  if (nvec <= 256) return launch_warp<BF16, ENTROPY, 16, 16>(a, rows, s);
  if (nvec <= 512) return launch_warp<BF16, ENTROPY, 16, 32>(a, rows, s);
  // vocabulary rows: a warp per row (K1d), split rows for small batches (K1e),
  // or (HS_CONF_IMPL=cta) K1b's CTA per row
  if (conf_impl() == 3) return launch_cta<BF16, ENTROPY, 256>(a, rows, s);
  cudaError_t e = cudaSuccess;
  if (launch_split<BF16, ENTROPY>(a, rows, s, &e)) return e;
  return launch_stream<BF16, ENTROPY>(a, rows, s);
}

}  // namespace

bool confidence_fusable(const ConfArgs& a) {
  // the dispatch below: rows of <= 128 x 16 B take the cp.async kernel (K1a)
  return a.L == 1 && a.nbatch == 1 && !a.late_wait && (a.top_k == 0 || (int64_t)a.top_k >= a.C) &&
         a.nvec <= 128 && conf_impl() == 2;
}

size_t split_ws_bytes(int64_t rows) {
  if (rows <= 0 || rows > kSplitMaxRows) return 0;
  return (size_t)kSplitMaxRows * sizeof(unsigned) + (size_t)rows * kSplitMaxSeg * sizeof(SplitPart);
}

const char* confidence_path(int64_t nvec) {
  if (nvec <= 512) return "warp-per-row";
  return conf_impl() == 3 ? "cta-per-row" : "warp-per-row-stream";
}

template <bool BF16, bool ENTROPY>
cudaError_t launch_topk(const ConfArgs& a, int64_t rows, cudaStream_t s) {
  auto k = conf_topk_kernel<BF16, ENTROPY>;
  constexpr size_t smem = (size_t)8 * kTopkPB * 32 * sizeof(float);
  static const int occ = [&] {
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    int b = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b, k, 256, smem);
    return b > 0 ? b : 1;
  }();
  const int64_t want = (rows + 7) / 8;
  const int64_t cap = (int64_t)num_sms() * occ;
  const int grid = (int)(want < cap ? (want > 0 ? want : 1) : cap);
  return launch_pdl(k, dim3(grid), dim3(256), smem, s, a);
}

cudaError_t launch_confidence(const ConfArgs& a, bool bf16, cudaStream_t s) {
  const int64_t rows = a.n * a.L * a.nbatch;
  const bool ent = a.kind == HS_CONF_ENTROPY || a.conf2 != nullptr;
  if (a.top_k > 0 && (int64_t)a.top_k < a.C) {
    if (bf16) return ent ? launch_topk<true, true>(a, rows, s) : launch_topk<true, false>(a, rows, s);
    return ent ? launch_topk<false, true>(a, rows, s) : launch_topk<false, false>(a, rows, s);
  }
  if (bf16) return ent ? dispatch<true, true>(a, rows, s) : dispatch<true, false>(a, rows, s);
  return ent ? dispatch<false, true>(a, rows, s) : dispatch<false, false>(a, rows, s);
}

cudaError_t launch_seq_reduce(const float* tok_conf, const uint8_t* tok_ok, int64_t n,
                              const int64_t* d_n, int L, int reduce, float* conf,
                              uint8_t* correct, cudaStream_t s) {
  const int64_t want = (n + 255) / 256;
  const int grid = (int)(want < 4096 ? (want > 0 ? want : 1) : 4096);
  return launch_pdl(seq_reduce_kernel, dim3(grid), dim3(256), 0, s, tok_conf, tok_ok, n, d_n, L,
                    reduce, conf, correct);
}

}  // namespace hs
