// api.cu -- the C-ABI of libhs.so (declared and documented in include/hs.h).
//
// Host side only: synchronous argument validation, workspace carving, variant
// selection and stream-ordered launches.  No allocation, no synchronisation.
#include <algorithm>
#include <atomic>
#include <cstdarg>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "hs_internal.h"

namespace hs {

static std::atomic<uint64_t> g_launches{0};
void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }
bool pdl_enabled() {
  static const bool on = [] {
    const char* e = getenv("HS_NO_PDL");
    return !(e && e[0] == '1');
  }();
  return on;
}

int num_sms() {
  static std::mutex mu;
  static std::vector<int> cache;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lk(mu);
  if ((int)cache.size() <= dev) cache.resize(dev + 1, 0);
  if (cache[dev] == 0) {
    int n = 0;
    cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    cache[dev] = n > 0 ? n : 1;
  }
  return cache[dev];
}

}  // namespace hs

namespace {

thread_local std::string g_err;

hs_status_t fail(hs_status_t s, const char* fmt, ...) __attribute__((format(printf, 2, 3)));
hs_status_t fail(hs_status_t s, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  return s;
}

hs_status_t cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess) return fail(HS_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
  return HS_OK;
}

inline bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }
inline size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

// workspace for hs_confidence with seq_len > 1: token conf (f32) + token ok (u8)
size_t conf_ws(int64_t n, int32_t L) {
  if (L <= 1) return 0;
  const size_t rows = (size_t)n * (size_t)L;
  return align_up(rows * sizeof(float), 256) + align_up(rows, 256);
}

hs_status_t check_logits(const void* logits, hs_dtype_t dtype, int64_t n, int32_t L, int64_t C,
                         int64_t stride, float T, hs_conf_kind_t kind, hs_seq_reduce_t reduce) {
  if (n < 0) return fail(HS_ERR_INVALID_ARGUMENT, "n = %lld < 0", (long long)n);
  if (dtype != HS_F32 && dtype != HS_BF16) return fail(HS_ERR_INVALID_ARGUMENT, "bad dtype %d", (int)dtype);
  if (C < 2) return fail(HS_ERR_INVALID_ARGUMENT, "n_classes = %lld < 2", (long long)C);
  if (L < 1) return fail(HS_ERR_INVALID_ARGUMENT, "seq_len = %d < 1", (int)L);
  if (stride < C) return fail(HS_ERR_INVALID_ARGUMENT, "row_stride %lld < n_classes %lld", (long long)stride, (long long)C);
  if (!(T > 0.f) || !std::isfinite(T)) return fail(HS_ERR_INVALID_ARGUMENT, "temperature must be > 0 and finite");
  if ((int)kind < 0 || (int)kind > 2) return fail(HS_ERR_INVALID_ARGUMENT, "bad confidence kind %d", (int)kind);
  if ((int)reduce < 0 || (int)reduce > 2) return fail(HS_ERR_INVALID_ARGUMENT, "bad seq reduce %d", (int)reduce);
  if (reduce == HS_SEQ_NONE && L != 1) return fail(HS_ERR_INVALID_ARGUMENT, "HS_SEQ_NONE requires seq_len == 1");
  const int eb = dtype == HS_BF16 ? 2 : 4;
  if (((stride * eb) & 15) != 0) return fail(HS_ERR_INVALID_ARGUMENT, "row_stride * element size must be a multiple of 16 bytes");
  if (n > 0 && (!logits || !aligned16(logits))) return fail(HS_ERR_INVALID_ARGUMENT, "logits must be non-NULL and 16-byte aligned");
  const int ve = 16 / eb;
  if ((C + ve - 1) / ve > (int64_t)0x7FFFFFFF / 8) return fail(HS_ERR_INVALID_ARGUMENT, "n_classes too large");
  return HS_OK;
}

hs::ConfArgs make_conf_args(const void* logits, hs_dtype_t dtype, int64_t n, int32_t L, int64_t C,
                            int64_t stride, const int64_t* row_index, const int64_t* d_n, float T,
                            hs_conf_kind_t kind) {
  hs::ConfArgs a{};
  const int eb = dtype == HS_BF16 ? 2 : 4, ve = 16 / eb;
  a.logits = logits;
  a.row_bytes = stride * eb;
  a.n = n;
  a.L = L;
  a.C = C;
  a.nvec = (int)((C + ve - 1) / ve);
  a.tail = (int)(C % ve);
  a.row_index = row_index;
  a.d_n = d_n;
  a.c = (float)(1.4426950408889634 / (double)T);
  a.kind = (int)kind;
  a.nbatch = 1;
  a.brows = n * L;
  return a;
}

// Runs K1 (+ K2) for prepared arguments (nbatch batches of n items).
hs_status_t run_confidence_args(hs::ConfArgs a, hs_dtype_t dtype, hs_seq_reduce_t reduce,
                                float* conf, int32_t* argmax, const int32_t* labels,
                                uint8_t* correct, void* ws, uint32_t* d_status, cudaStream_t s) {
  const int64_t n = a.n;
  const int32_t L = a.L;
  const int64_t items = n * a.nbatch;
  const int64_t* d_n = a.d_n;
  a.argmax = argmax;
  a.labels = labels;
  a.status = d_status;
  if (L == 1) {
    a.conf = conf;
    a.ok = correct;
    return cuda_check(hs::launch_confidence(a, dtype == HS_BF16, s), "confidence kernel");
  }
  float* tok_conf = reinterpret_cast<float*>(ws);
  uint8_t* tok_ok = reinterpret_cast<uint8_t*>(ws) + align_up((size_t)items * L * sizeof(float), 256);
  a.conf = tok_conf;
  a.ok = (correct && labels) ? tok_ok : nullptr;
  hs_status_t st = cuda_check(hs::launch_confidence(a, dtype == HS_BF16, s), "confidence kernel");
  if (st != HS_OK) return st;
  return cuda_check(hs::launch_seq_reduce(tok_conf, a.ok, items, a.nbatch == 1 ? d_n : nullptr, L,
                                          (int)reduce, conf, correct, s),
                    "sequence reduce kernel");
}

hs_status_t run_confidence(const void* logits, hs_dtype_t dtype, int64_t n, int32_t L, int64_t C,
                           int64_t stride, const int64_t* row_index, const int64_t* d_n, float T,
                           hs_conf_kind_t kind, hs_seq_reduce_t reduce, float* conf,
                           int32_t* argmax, const int32_t* labels, uint8_t* correct, void* ws,
                           uint32_t* d_status, cudaStream_t s) {
  if (n == 0) return HS_OK;
  hs::ConfArgs a = make_conf_args(logits, dtype, n, L, C, stride, row_index, d_n, T, kind);
  return run_confidence_args(a, dtype, reduce, conf, argmax, labels, correct, ws, d_status, s);
}

hs_status_t check_threshold(float t) {
  if (std::isnan(t) || (t < 0.f) || (t > 1.f && !std::isinf(t)))
    return fail(HS_ERR_INVALID_ARGUMENT, "threshold must be in [0,1] or +inf");
  return HS_OK;
}

}  // namespace

extern "C" {

const char* hs_status_string(hs_status_t s) {
  switch (s) {
    case HS_OK: return "HS_OK";
    case HS_ERR_INVALID_ARGUMENT: return "HS_ERR_INVALID_ARGUMENT";
    case HS_ERR_NONFINITE_INPUT: return "HS_ERR_NONFINITE_INPUT";
    case HS_ERR_CUDA: return "HS_ERR_CUDA";
    case HS_ERR_NCCL: return "HS_ERR_NCCL";
    case HS_ERR_WORKSPACE_TOO_SMALL: return "HS_ERR_WORKSPACE_TOO_SMALL";
    case HS_ERR_UNSUPPORTED: return "HS_ERR_UNSUPPORTED";
  }
  return "HS_ERR_UNKNOWN";
}

const char* hs_last_error(void) { return g_err.c_str(); }
uint64_t hs_launch_count(void) { return hs::g_launches.load(); }
const char* hs_build_info(void) {
#define HS_STR2(x) #x
#define HS_STR(x) HS_STR2(x)
#if defined(HS_EXP_NOARGMAX) || defined(HS_EXP_NOEXP) || defined(HS_EXP_TOPK_NOCAND) || \
    defined(HS_EXP_FZ_NOSYNC) || defined(HS_EXP_FZ_NOFINISH)
  // timing-bound experiment build (tools/build_variants.py): results are WRONG;
  // the Python loader refuses it unless HS_ALLOW_EXPERIMENT=1
  return "libhs: sm_100a (compute_100a), nvcc " HS_STR(__CUDACC_VER_MAJOR__) "." HS_STR(__CUDACC_VER_MINOR__)
         " EXPERIMENT-WRONG-RESULTS";
#else
  return "libhs: sm_100a (compute_100a), nvcc " HS_STR(__CUDACC_VER_MAJOR__) "." HS_STR(__CUDACC_VER_MINOR__);
#endif
}

// mandatory part (token rows of sequences) + the optional split-row region
size_t hs_confidence_workspace(int64_t n, int32_t seq_len) {
  if (n < 0) n = 0;
  const size_t split = hs::split_ws_bytes(n * (int64_t)(seq_len < 1 ? 1 : seq_len));
  return split ? align_up(conf_ws(n, seq_len), 256) + split : conf_ws(n, seq_len);
}

hs_status_t hs_confidence(const void* logits, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                          int64_t n_classes, int64_t row_stride, const int64_t* row_index,
                          const int64_t* d_n, float temperature, hs_conf_kind_t kind,
                          hs_seq_reduce_t reduce, float* conf, int32_t* argmax,
                          const int32_t* labels, uint8_t* correct, void* ws, size_t ws_bytes,
                          uint32_t* d_status, hs_stream_t stream) {
  return hs_confidence_topk(logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n,
                            temperature, kind, reduce, 0, conf, argmax, labels, correct, ws,
                            ws_bytes, d_status, stream);
}

hs_status_t hs_confidence_topk(const void* logits, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                               int64_t n_classes, int64_t row_stride, const int64_t* row_index,
                               const int64_t* d_n, float temperature, hs_conf_kind_t kind,
                               hs_seq_reduce_t reduce, int32_t top_k, float* conf, int32_t* argmax,
                               const int32_t* labels, uint8_t* correct, void* ws, size_t ws_bytes,
                               uint32_t* d_status, hs_stream_t stream) {
  return hs_confidence_ex(logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n, temperature,
                          kind, reduce, top_k, conf, nullptr, argmax, labels, correct, ws, ws_bytes,
                          d_status, stream);
}

hs_status_t hs_confidence_ex(const void* logits, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                             int64_t n_classes, int64_t row_stride, const int64_t* row_index,
                             const int64_t* d_n, float temperature, hs_conf_kind_t kind,
                             hs_seq_reduce_t reduce, int32_t top_k, float* conf, float* conf_entropy,
                             int32_t* argmax, const int32_t* labels, uint8_t* correct, void* ws,
                             size_t ws_bytes, uint32_t* d_status, hs_stream_t stream) {
  hs_status_t st = check_logits(logits, dtype, n, seq_len, n_classes, row_stride, temperature, kind, reduce);
  if (st == HS_OK && conf_entropy && seq_len != 1)
    st = fail(HS_ERR_INVALID_ARGUMENT, "conf_entropy requires seq_len == 1");
  if (st != HS_OK) return st;
  if (top_k < 0 || top_k > hs::kTopkMax)
    return fail(HS_ERR_INVALID_ARGUMENT, "top_k = %d outside 0..%d", top_k, hs::kTopkMax);
  if (n > 0 && !conf) return fail(HS_ERR_INVALID_ARGUMENT, "conf output is required");
  if (correct && !labels) return fail(HS_ERR_INVALID_ARGUMENT, "correct requires labels");
  if (ws_bytes < conf_ws(n, seq_len) || (conf_ws(n, seq_len) && !ws))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, conf_ws(n, seq_len));
  if (n == 0) return HS_OK;
  hs::ConfArgs a = make_conf_args(logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n,
                                  temperature, kind);
  a.top_k = top_k;
  a.conf2 = conf_entropy;
  {  // optional split-row region: used when the caller's workspace has room for it;
     // its arrival counters are zeroed by the launcher (no zero-fill contract here)
    const size_t base = align_up(conf_ws(n, seq_len), 256);
    const size_t split = hs::split_ws_bytes(n * (int64_t)seq_len);
    if (split && ws && ws_bytes >= base + split) {
      a.split_ws = reinterpret_cast<char*>(ws) + base;
      a.split_zero = 1;
    }
  }
  return run_confidence_args(a, dtype, reduce, conf, argmax, labels, correct, ws, d_status,
                             (cudaStream_t)stream);
}

size_t hs_confidence_batched_workspace(int32_t n_batches, int64_t n, int32_t seq_len) {
  return conf_ws((int64_t)(n_batches < 1 ? 1 : n_batches) * n, seq_len);
}

hs_status_t hs_confidence_batched(const void* const* logits, const float* temperatures,
                                  int32_t n_batches, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                                  int64_t n_classes, int64_t row_stride,
                                  const int64_t* row_index, hs_conf_kind_t kind,
                                  hs_seq_reduce_t reduce, float* conf, int32_t* argmax,
                                  const int32_t* labels, uint8_t* correct, void* ws,
                                  size_t ws_bytes, uint32_t* d_status, hs_stream_t stream) {
  if (!logits || !temperatures) return fail(HS_ERR_INVALID_ARGUMENT, "logits/temperatures arrays are required");
  if (n_batches < 1 || n_batches > hs::kMaxBatch)
    return fail(HS_ERR_INVALID_ARGUMENT, "n_batches = %d outside 1..%d", n_batches, hs::kMaxBatch);
  for (int b = 0; b < n_batches; ++b) {
    hs_status_t st = check_logits(logits[b], dtype, n, seq_len, n_classes, row_stride,
                                  temperatures[b], kind, reduce);
    if (st != HS_OK) return st;
  }
  if (n > 0 && !conf) return fail(HS_ERR_INVALID_ARGUMENT, "conf output is required");
  if (correct && !labels) return fail(HS_ERR_INVALID_ARGUMENT, "correct requires labels");
  if ((int64_t)n_batches * n * seq_len >= (int64_t(1) << 32))
    return fail(HS_ERR_INVALID_ARGUMENT, "n_batches * n * seq_len must be < 2^32");
  const size_t need = conf_ws((int64_t)n_batches * n, seq_len);
  if (ws_bytes < need || (need && !ws))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
  if (n == 0) return HS_OK;
  hs::ConfArgs a = make_conf_args(logits[0], dtype, n, seq_len, n_classes, row_stride, row_index,
                                  nullptr, temperatures[0], kind);
  a.nbatch = n_batches;
  a.brows = n * seq_len;
  // exact for every row < 2^32: (2^64 + e) / d with e < d, row * e < 2^64
  a.bmagic = a.brows >= 2 ? (uint64_t)(~0ull / (uint64_t)a.brows) + 1ull : 0ull;
  for (int b = 0; b < n_batches; ++b) {
    a.bptr[b] = logits[b];
    a.bc[b] = (float)(1.4426950408889634 / (double)temperatures[b]);
  }
  return run_confidence_args(a, dtype, reduce, conf, argmax, labels, correct, ws, d_status,
                             (cudaStream_t)stream);
}

size_t hs_fit_temperature_workspace(int32_t n_batches, int64_t n) {
  return hs::temp_fit_ws_bytes(n_batches < 1 ? 1 : n_batches, n);
}

hs_status_t hs_fit_temperature(const void* const* logits, int32_t n_batches, hs_dtype_t dtype,
                               int64_t n, int64_t n_classes, int64_t row_stride,
                               const int32_t* labels, double t_lo, double t_hi, int32_t max_passes,
                               float* d_T, double* d_nll, int32_t* d_passes, int64_t* d_used,
                               void* ws, size_t ws_bytes, uint32_t* d_status, hs_stream_t stream) {
  if (!logits) return fail(HS_ERR_INVALID_ARGUMENT, "logits array is required");
  if (n_batches < 1 || n_batches > hs::kMaxBatch)
    return fail(HS_ERR_INVALID_ARGUMENT, "n_batches = %d outside 1..%d", n_batches, hs::kMaxBatch);
  for (int b = 0; b < n_batches; ++b) {
    hs_status_t st = check_logits(logits[b], dtype, n, 1, n_classes, row_stride, 1.0f,
                                  HS_CONF_MAXPROB, HS_SEQ_NONE);
    if (st != HS_OK) return st;
  }
  if (!(t_lo > 0.0) || !(t_lo <= t_hi) || !std::isfinite(t_hi))
    return fail(HS_ERR_INVALID_ARGUMENT, "temperature range must satisfy 0 < t_lo <= t_hi < inf");
  if (max_passes < 1 || max_passes > 256)
    return fail(HS_ERR_INVALID_ARGUMENT, "max_passes = %d outside 1..256", max_passes);
  if (!d_T) return fail(HS_ERR_INVALID_ARGUMENT, "d_T output is required");
  if (n > 0 && !labels) return fail(HS_ERR_INVALID_ARGUMENT, "labels are required");
  const size_t need = hs::temp_fit_ws_bytes(n_batches, n);
  if (ws_bytes < need || !ws) return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
  hs::TfArgs a{};
  const int eb = dtype == HS_BF16 ? 2 : 4, ve = 16 / eb;
  for (int b = 0; b < n_batches; ++b) a.bptr[b] = logits[b];
  a.nbatch = n_batches;
  a.n = n;
  a.row_bytes = row_stride * eb;
  a.C = n_classes;
  a.nvec = (int)((n_classes + ve - 1) / ve);
  a.tail = (int)(n_classes % ve);
  a.labels = labels;
  a.blo0 = 1.0 / t_hi;
  a.bhi0 = 1.0 / t_lo;
  a.t_lo = t_lo;
  a.t_hi = t_hi;
  a.tol = 1.0 / (double)(1 << 21);
  a.max_passes = max_passes;
  a.T = d_T;
  a.nll = d_nll;
  a.passes = d_passes;
  a.used = d_used;
  a.status = d_status;
  return cuda_check(hs::launch_temp_fit(a, dtype == HS_BF16, ws, (cudaStream_t)stream),
                    "temperature fitting kernel");
}

int64_t hs_grid_size(int32_t K, int32_t log2_bins) {
  if (K < 2 || K > hs::kReplayMaxK || log2_bins < 1 || log2_bins > 14) return -1;
  const int64_t R = ((int64_t)1 << log2_bins) + 2;
  int64_t S = 1;
  for (int k = 0; k < K - 1; ++k) {
    S *= R;
    if (S >= ((int64_t)1 << 31)) return -1;
  }
  return S;
}

hs_status_t hs_grid_vector(int64_t s, int32_t K, int32_t log2_bins, int32_t* b) {
  const int64_t S = hs_grid_size(K, log2_bins);
  if (S < 0 || s < 0 || s >= S || !b) return fail(HS_ERR_INVALID_ARGUMENT, "bad grid vector query");
  const int64_t R = ((int64_t)1 << log2_bins) + 2;
  for (int k = K - 2; k >= 0; --k) {
    b[k] = (int32_t)(s % R);
    s /= R;
  }
  return HS_OK;
}

size_t hs_threshold_replay_workspace(int32_t K, int64_t N, int32_t log2_bins) {
  if (K < 2 || K > hs::kReplayMaxK || log2_bins < 1 || log2_bins > 14) return 0;
  return hs::replay_ws_bytes(K, N < 0 ? 0 : N, log2_bins);
}

hs_status_t hs_threshold_replay(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                int32_t log2_bins, const int32_t* d_bvecs, int64_t S,
                                const int64_t* weights, int64_t* d_correct, int64_t* d_energy,
                                int64_t* d_reach, int64_t* d_model_correct, void* ws,
                                size_t ws_bytes, hs_stream_t stream) {
  if (K < 2 || K > hs::kReplayMaxK) return fail(HS_ERR_INVALID_ARGUMENT, "K = %d outside 2..%d", K, hs::kReplayMaxK);
  if (log2_bins < 1 || log2_bins > 14) return fail(HS_ERR_INVALID_ARGUMENT, "log2_bins = %d outside 1..14", log2_bins);
  if (N < 1 || N >= ((int64_t)1 << 32)) return fail(HS_ERR_INVALID_ARGUMENT, "N = %lld outside 1..2^32-1 (empty trace)", (long long)N);
  if (S < 0 || S >= ((int64_t)1 << 31)) return fail(HS_ERR_INVALID_ARGUMENT, "S = %lld outside 0..2^31-1", (long long)S);
  if (!d_bvecs && S != hs_grid_size(K, log2_bins))
    return fail(HS_ERR_INVALID_ARGUMENT, "d_bvecs == NULL requires S == hs_grid_size(K, log2_bins)");
  if (!conf || !correct || !weights || (S > 0 && (!d_correct || !d_energy)))
    return fail(HS_ERR_INVALID_ARGUMENT, "conf, correct, weights, d_correct and d_energy are required");
  hs::ReplayArgs a{};
  unsigned long long cum = 0;
  for (int k = 0; k < K; ++k) {
    if (weights[k] < 0) return fail(HS_ERR_INVALID_ARGUMENT, "weights must be >= 0");
    const unsigned long long add = (unsigned long long)weights[k];
    if (cum + add < cum || (cum + add) > (~0ull >> 1) / (unsigned long long)N)
      return fail(HS_ERR_INVALID_ARGUMENT, "energy would overflow int64");
    cum += add;
    a.w.cum[k] = cum;
  }
  const size_t need = hs::replay_ws_bytes(K, N, log2_bins);
  if (ws_bytes < need || !ws) return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
  a.K = K;
  a.N = N;
  a.q = log2_bins;
  a.bvecs = d_bvecs;
  a.S = S;
  a.out_c = d_correct;
  a.out_e = d_energy;
  a.reach = d_reach;
  return cuda_check(hs::launch_replay(a, conf, correct, reinterpret_cast<unsigned long long*>(d_model_correct),
                                      ws, (cudaStream_t)stream),
                    "threshold replay kernels");
}

size_t hs_perf_graph_workspace(int64_t N) { return hs::graph_ws_bytes(N < 0 ? 0 : N); }

hs_status_t hs_perf_graph(const int64_t* d_correct, const int64_t* d_energy, int64_t S, int64_t N,
                          int64_t tau, int64_t floor_, const int64_t* d_model_correct, int32_t K,
                          int64_t* d_front_c, int64_t* d_front_e, int64_t* d_front_s,
                          int64_t* d_front_n, int64_t* d_pick, void* ws, size_t ws_bytes,
                          uint32_t* d_status, hs_stream_t stream) {
  if (S < 0 || N < 0) return fail(HS_ERR_INVALID_ARGUMENT, "S and N must be >= 0");
  if (S > 0 && (!d_correct || !d_energy)) return fail(HS_ERR_INVALID_ARGUMENT, "d_correct / d_energy are required");
  if (!d_front_c || !d_front_e || !d_front_s || !d_front_n || !d_pick)
    return fail(HS_ERR_INVALID_ARGUMENT, "frontier outputs and d_pick are required");
  if ((tau < 0 || floor_ < 0) && (!d_model_correct || K < 2 || K > hs::kReplayMaxK))
    return fail(HS_ERR_INVALID_ARGUMENT, "tau / floor < 0 need d_model_correct and 2 <= K <= %d", hs::kReplayMaxK);
  const size_t need = hs::graph_ws_bytes(N);
  if (ws_bytes < need || !ws) return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
  return cuda_check(hs::launch_graph(d_correct, d_energy, S, N, tau, floor_,
                                     reinterpret_cast<const unsigned long long*>(d_model_correct), K,
                                     d_front_c, d_front_e, d_front_s, d_front_n, d_pick, d_status, ws,
                                     (cudaStream_t)stream),
                    "performance graph kernels");
}

// ---- multi-GPU group over peer memory (peer.cu) -------------------------------
static hs_status_t peer_args(const hs_peer_t* g, bool need_pay, hs::PeerArgs* out, hs::PeerLayout* lay) {
  if (!g) return fail(HS_ERR_INVALID_ARGUMENT, "peer group is required");
  if (g->world < 1 || g->world > hs::kPeerMaxWorld || g->rank < 0 || g->rank >= g->world)
    return fail(HS_ERR_INVALID_ARGUMENT, "rank %d / world %d out of range", g->rank, g->world);
  if (g->cap < 0 || g->cap >= ((int64_t)1 << 32) || g->payload_row_bytes < 0 || (g->payload_row_bytes % 16) ||
      g->log2_bins < 1 || g->log2_bins > 14)
    return fail(HS_ERR_INVALID_ARGUMENT, "0 <= cap < 2^32, payload_row_bytes %% 16 == 0 and 1 <= log2_bins <= 14");
  if (need_pay && g->payload_row_bytes == 0)
    return fail(HS_ERR_INVALID_ARGUMENT, "the group's regions were sized without payload rows");
  const hs::PeerLayout L = hs::peer_layout(g->world, g->cap, g->payload_row_bytes, g->log2_bins);
  hs::PeerArgs A{};
  A.world = g->world;
  A.rank = g->rank;
  A.recv_stride = (int64_t)L.recv_stride;
  for (int h = 0; h < g->world; ++h) {
    char* r = reinterpret_cast<char*>(g->region[h]);
    if (!r || !aligned16(r)) return fail(HS_ERR_INVALID_ARGUMENT, "region[%d] is NULL or misaligned", h);
    A.hdr[h] = reinterpret_cast<hs::PeerHeader*>(r);
    A.recv_ids[h] = reinterpret_cast<int64_t*>(r + L.recv_off);
    A.recv_payload[h] = g->payload_row_bytes ? r + L.pay_off : nullptr;
  }
  *out = A;
  if (lay) *lay = L;
  return HS_OK;
}

static hs_status_t peer_dest(const hs_peer_t* g, const int32_t* dest_ranks, int32_t n_dest, hs::PeerDest* d) {
  if (!dest_ranks) {     // NULL: every rank, in rank order (the balanced placement)
    d->n = g->world;
    for (int i = 0; i < g->world; ++i) d->ranks[i] = i;
    return HS_OK;
  }
  if (n_dest < 1 || n_dest > g->world) return fail(HS_ERR_INVALID_ARGUMENT, "1 <= n_dest <= world");
  d->n = n_dest;
  unsigned seen = 0;
  for (int i = 0; i < n_dest; ++i) {
    if (dest_ranks[i] < 0 || dest_ranks[i] >= g->world || (seen >> dest_ranks[i]) & 1u)
      return fail(HS_ERR_INVALID_ARGUMENT, "dest_ranks must be distinct ranks of the group");
    seen |= 1u << dest_ranks[i];
    d->ranks[i] = dest_ranks[i];
  }
  return HS_OK;
}

size_t hs_peer_region_bytes(int32_t world, int64_t cap, int64_t payload_row_bytes, int32_t log2_bins) {
  if (world < 1 || world > hs::kPeerMaxWorld || cap < 0 || payload_row_bytes < 0 || log2_bins < 1 ||
      log2_bins > 14)
    return 0;
  return hs::peer_layout(world, cap, payload_row_bytes, log2_bins).bytes;
}

int64_t* hs_peer_recv_ids(const hs_peer_t* g, int32_t set) {
  hs::PeerArgs A;
  if (set < 0 || set > 1 || peer_args(g, false, &A, nullptr) != HS_OK) return nullptr;
  return A.recv_ids[g->rank] + (int64_t)set * A.recv_stride;
}

void* hs_peer_recv_payload(const hs_peer_t* g, int32_t set) {
  hs::PeerArgs A;
  if (set < 0 || set > 1 || peer_args(g, false, &A, nullptr) != HS_OK || !g->payload_row_bytes) return nullptr;
  return reinterpret_cast<char*>(A.recv_payload[g->rank]) + (int64_t)set * A.recv_stride * g->payload_row_bytes;
}

hs_status_t hs_peer_forward_publish(const hs_peer_t* g, const int64_t* d_count, uint32_t* d_status,
                                    hs_stream_t stream) {
  hs::PeerArgs A;
  hs_status_t st = peer_args(g, false, &A, nullptr);
  if (st != HS_OK) return st;
  if (!d_count) return fail(HS_ERR_INVALID_ARGUMENT, "d_count is required");
  return cuda_check(hs::launch_peer_publish(d_count, g->cap, A, d_status, (cudaStream_t)stream),
                    "peer publish kernel");
}

hs_status_t hs_peer_forward_scatter(const hs_peer_t* g, int32_t set, const int64_t* ids, const void* payload,
                                    const int32_t* dest_ranks, int32_t n_dest, int64_t* d_recv_count,
                                    uint32_t* d_status, hs_stream_t stream) {
  hs::PeerArgs A;
  hs_status_t st = peer_args(g, payload != nullptr, &A, nullptr);
  if (st != HS_OK) return st;
  if (set < 0 || set > 1) return fail(HS_ERR_INVALID_ARGUMENT, "set must be 0 or 1");
  if (!ids || !d_recv_count) return fail(HS_ERR_INVALID_ARGUMENT, "ids and d_recv_count are required");
  if (payload && !aligned16(payload)) return fail(HS_ERR_INVALID_ARGUMENT, "payload must be 16-byte aligned");
  hs::PeerDest d{};
  st = peer_dest(g, dest_ranks, n_dest, &d);
  if (st != HS_OK) return st;
  return cuda_check(hs::launch_peer_scatter(ids, payload, payload ? g->payload_row_bytes : 0, g->cap, set, A,
                                            d, d_recv_count, d_status, (cudaStream_t)stream),
                    "peer scatter kernel");
}

hs_status_t hs_peer_forward_wait(const hs_peer_t* g, uint32_t* d_status, hs_stream_t stream) {
  hs::PeerArgs A;
  hs_status_t st = peer_args(g, false, &A, nullptr);
  if (st != HS_OK) return st;
  return cuda_check(hs::launch_peer_wait(A, d_status, (cudaStream_t)stream), "peer wait kernel");
}

hs_status_t hs_peer_forward(const hs_peer_t* g, int32_t set, const int64_t* ids, const void* payload,
                            const int64_t* d_count, const int32_t* dest_ranks, int32_t n_dest,
                            int64_t* d_recv_count, uint32_t* d_status, hs_stream_t stream) {
  // validate everything first: a rank that fails after publishing would leave
  // its peers waiting (they time out instead of hanging, but still)
  hs::PeerArgs A;
  hs_status_t st = peer_args(g, payload != nullptr, &A, nullptr);
  if (st != HS_OK) return st;
  hs::PeerDest d{};
  st = peer_dest(g, dest_ranks, n_dest, &d);
  if (st != HS_OK) return st;
  if (set < 0 || set > 1 || !ids || !d_count || !d_recv_count || (payload && !aligned16(payload)))
    return fail(HS_ERR_INVALID_ARGUMENT, "set in {0,1}, ids, d_count, d_recv_count (aligned payload) required");
  st = hs_peer_forward_publish(g, d_count, d_status, stream);
  if (st == HS_OK) st = hs_peer_forward_scatter(g, set, ids, payload, dest_ranks, n_dest, d_recv_count, d_status, stream);
  if (st == HS_OK) st = hs_peer_forward_wait(g, d_status, stream);
  return st;
}

hs_status_t hs_ipc_alloc(size_t bytes, void** dptr) {
  if (!dptr || bytes == 0) return fail(HS_ERR_INVALID_ARGUMENT, "dptr and bytes > 0 are required");
  hs_status_t st = cuda_check(cudaMalloc(dptr, bytes), "cudaMalloc");
  if (st != HS_OK) return st;
  st = cuda_check(cudaMemset(*dptr, 0, bytes), "cudaMemset");
  if (st == HS_OK) st = cuda_check(cudaDeviceSynchronize(), "cudaDeviceSynchronize");
  return st;
}

hs_status_t hs_ipc_free(void* dptr) {
  if (!dptr) return fail(HS_ERR_INVALID_ARGUMENT, "dptr is required");
  return cuda_check(cudaFree(dptr), "cudaFree");
}

hs_status_t hs_ipc_handle(const void* dptr, void* handle) {
  static_assert(sizeof(cudaIpcMemHandle_t) == 64, "IPC handle size");
  if (!dptr || !handle) return fail(HS_ERR_INVALID_ARGUMENT, "dptr and handle are required");
  cudaIpcMemHandle_t h;
  hs_status_t st = cuda_check(cudaIpcGetMemHandle(&h, const_cast<void*>(dptr)), "cudaIpcGetMemHandle");
  if (st == HS_OK) memcpy(handle, &h, sizeof h);
  return st;
}

hs_status_t hs_ipc_open(const void* handle, void** dptr) {
  if (!handle || !dptr) return fail(HS_ERR_INVALID_ARGUMENT, "handle and dptr are required");
  cudaIpcMemHandle_t h;
  memcpy(&h, handle, sizeof h);
  return cuda_check(cudaIpcOpenMemHandle(dptr, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
}

hs_status_t hs_ipc_close(void* dptr) {
  if (!dptr) return fail(HS_ERR_INVALID_ARGUMENT, "dptr is required");
  return cuda_check(cudaIpcCloseMemHandle(dptr), "cudaIpcCloseMemHandle");
}

hs_status_t hs_comm_unique_id(void* id) {
  if (!id) return fail(HS_ERR_INVALID_ARGUMENT, "id is required");
  if (!hs::nccl_available()) return fail(HS_ERR_UNSUPPORTED, "libnccl.so.2 could not be loaded");
  const int r = hs::nccl_unique_id(id);
  return r ? fail(HS_ERR_NCCL, "ncclGetUniqueId: %s", hs::nccl_error(r)) : HS_OK;
}

hs_status_t hs_comm_create(const void* id, int32_t rank, int32_t world, int32_t device, hs_comm_t* out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world || device < 0)
    return fail(HS_ERR_INVALID_ARGUMENT, "id, out, 0 <= rank < world and device >= 0 are required");
  if (!hs::nccl_available()) return fail(HS_ERR_UNSUPPORTED, "libnccl.so.2 could not be loaded");
  const int r = hs::nccl_comm_create(id, rank, world, device, out);
  return r ? fail(HS_ERR_NCCL, "ncclCommInitRank: %s", hs::nccl_error(r)) : HS_OK;
}

hs_status_t hs_comm_destroy(hs_comm_t comm) {
  if (!comm) return fail(HS_ERR_INVALID_ARGUMENT, "comm is required");
  const int r = hs::nccl_comm_destroy(comm);
  return r ? fail(HS_ERR_NCCL, "ncclCommDestroy: %s", hs::nccl_error(r)) : HS_OK;
}

static hs_status_t check_calib(int32_t K, int32_t q, void* ws, size_t ws_bytes);

hs_status_t hs_calibrate_thresholds_comm(const float* conf, const uint8_t* correct, int32_t K,
                                         int64_t N, int32_t log2_bins, int64_t target_correct,
                                         int32_t* d_bin_idx, float* d_thresholds, int64_t* d_reach,
                                         int64_t* d_handled, int64_t* d_correct_total,
                                         hs_comm_t comm, void* ws, size_t ws_bytes,
                                         hs_stream_t stream) {
  return hs_calibrate_thresholds_comm_ex(conf, correct, K, N, log2_bins, target_correct, 0, d_bin_idx,
                                         d_thresholds, d_reach, d_handled, d_correct_total, comm, ws,
                                         ws_bytes, stream);
}

hs_status_t hs_calibrate_thresholds_comm_ex(const float* conf, const uint8_t* correct, int32_t K,
                                            int64_t N, int32_t log2_bins, int64_t target_correct,
                                            int32_t refine_passes, int32_t* d_bin_idx, float* d_thresholds,
                                            int64_t* d_reach, int64_t* d_handled, int64_t* d_correct_total,
                                            hs_comm_t comm, void* ws, size_t ws_bytes, hs_stream_t stream) {
  if (refine_passes < 0 || refine_passes > 64)
    return fail(HS_ERR_INVALID_ARGUMENT, "refine_passes = %d outside 0..64", refine_passes);
  if (!d_bin_idx || !d_thresholds || !d_reach || !d_handled || !d_correct_total)
    return fail(HS_ERR_INVALID_ARGUMENT, "all calibration outputs are required");
  // validate everything the rounds will check before any collective is posted
  hs_status_t st = check_calib(K, log2_bins, ws, ws_bytes);
  if (st != HS_OK) return st;
  if (N < 0) return fail(HS_ERR_INVALID_ARGUMENT, "N < 0");
  if (N > 0 && (!conf || !correct)) return fail(HS_ERR_INVALID_ARGUMENT, "NULL input");
  st = hs_calibrate_begin(K, log2_bins, target_correct, ws, ws_bytes, stream);
  if (st != HS_OK) return st;
  int32_t* hist = hs_calibrate_hist_ptr(ws);
  const size_t words = hs_calibrate_hist_bytes(log2_bins) / sizeof(int32_t);
  for (int32_t k = 0; k < K - 1; ++k) {
    st = hs_calibrate_histogram(conf, correct, K, N, log2_bins, k, d_bin_idx, ws, ws_bytes, stream);
    if (st != HS_OK) return st;
    if (comm) {
      const int r = hs::nccl_allreduce_i32_sum(hist, words, comm, (cudaStream_t)stream);
      if (r) return fail(HS_ERR_NCCL, "ncclAllReduce: %s", hs::nccl_error(r));
    }
    st = hs_calibrate_select(K, log2_bins, k, d_bin_idx, d_thresholds, d_reach, d_handled,
                             d_correct_total, ws, ws_bytes, stream);
    if (st != HS_OK) return st;
  }
  if (refine_passes == 0) return HS_OK;
  // D5 refinement on the sharded set: per pass and stage, each rank histograms
  // its samples that reach k (downstream correctness as third channel) and adds
  // A_k (answers given before k); histogram and A_k are summed across ranks,
  // every rank selects the same b_k; a final replay's counts are summed too.
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* d_A = reinterpret_cast<int64_t*>(ws);     // CalibState::A (first field)
  for (int32_t p = 0; p < refine_passes; ++p) {
    for (int32_t k = 0; k < K - 1; ++k) {
      st = cuda_check(hs::launch_calib_refine_round(conf, correct, K, N, log2_bins, k, d_bin_idx, ws, p == 0 && k == 0, s),
                      "calib refinement histogram");
      if (st != HS_OK) return st;
      if (comm) {
        int r = hs::nccl_allreduce_i32_sum(hist, words, comm, s);
        if (!r) r = hs::nccl_allreduce_i64_sum(d_A, 1, comm, s);
        if (r) return fail(HS_ERR_NCCL, "ncclAllReduce (refinement): %s", hs::nccl_error(r));
      }
      st = hs_calibrate_select(K, log2_bins, k, d_bin_idx, d_thresholds, d_reach, d_handled, d_correct_total,
                               ws, ws_bytes, stream);
      if (st != HS_OK) return st;
    }
  }
  st = cuda_check(hs::launch_calib_replay(conf, correct, K, N, log2_bins, d_bin_idx, d_reach, d_handled,
                                          d_correct_total, s),
                  "calib replay");
  if (st != HS_OK || !comm) return st;
  int r = hs::nccl_allreduce_i64_sum(d_reach, K, comm, s);
  if (!r) r = hs::nccl_allreduce_i64_sum(d_handled, K, comm, s);
  if (!r) r = hs::nccl_allreduce_i64_sum(d_correct_total, 1, comm, s);
  return r ? fail(HS_ERR_NCCL, "ncclAllReduce (replay): %s", hs::nccl_error(r)) : HS_OK;
}

// ws: this rank's (count, recv_cap) pair, then every rank's pairs
size_t hs_forward_nccl_workspace(int32_t world) { return (size_t)(2 + 2 * (world < 1 ? 1 : world)) * sizeof(int64_t) + 256; }

hs_status_t hs_forward_nccl(const int64_t* ids, const void* payload, int64_t payload_row_bytes,
                            const int64_t* d_count, const int32_t* dest_ranks, int32_t n_dest,
                            int64_t* recv_ids, void* recv_payload, int64_t recv_cap,
                            int64_t* h_recv_count, hs_comm_t comm, void* ws, size_t ws_bytes,
                            hs_stream_t stream) {
  if (!comm) return fail(HS_ERR_INVALID_ARGUMENT, "comm is required");
  const int W = hs::nccl_world(comm), rank = hs::nccl_rank(comm);
  if (!ids || !d_count || !recv_ids || !h_recv_count || recv_cap < 0)
    return fail(HS_ERR_INVALID_ARGUMENT, "ids, d_count, recv_ids and h_recv_count are required");
  if (payload_row_bytes < 0 || (payload_row_bytes && (!payload || !recv_payload)))
    return fail(HS_ERR_INVALID_ARGUMENT, "payload buffers are required when payload_row_bytes > 0");
  if (!dest_ranks || n_dest < 1 || n_dest > W) return fail(HS_ERR_INVALID_ARGUMENT, "1 <= n_dest <= world");
  std::vector<int> is_dest(W, -1);
  for (int i = 0; i < n_dest; ++i) {
    if (dest_ranks[i] < 0 || dest_ranks[i] >= W || is_dest[dest_ranks[i]] >= 0)
      return fail(HS_ERR_INVALID_ARGUMENT, "dest_ranks must be distinct ranks of the group");
    is_dest[dest_ranks[i]] = i;
  }
  if (!ws || ws_bytes < hs_forward_nccl_workspace(W))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, hs_forward_nccl_workspace(W));
  cudaStream_t s = (cudaStream_t)stream;
  int64_t* d_mine = reinterpret_cast<int64_t*>(ws);
  int64_t* d_all = d_mine + 2;
  // every rank learns every rank's (count, recv_cap): the capacity check below
  // is then the same decision on all ranks, taken before any send/recv is posted
  hs_status_t st = cuda_check(cudaMemcpyAsync(d_mine, d_count, sizeof(int64_t), cudaMemcpyDeviceToDevice, s),
                              "count copy");
  if (st == HS_OK)
    st = cuda_check(cudaMemcpyAsync(d_mine + 1, &recv_cap, sizeof(int64_t), cudaMemcpyHostToDevice, s),
                    "capacity copy");
  if (st != HS_OK) return st;
  int r = hs::nccl_allgather_i64(d_mine, d_all, 2, comm, s);
  if (r) return fail(HS_ERR_NCCL, "ncclAllGather: %s", hs::nccl_error(r));
  std::vector<int64_t> pairs(2 * W), cnt(W), caps(W);
  st = cuda_check(cudaMemcpyAsync(pairs.data(), d_all, 2 * W * sizeof(int64_t), cudaMemcpyDeviceToHost, s),
                  "count read-back");
  if (st == HS_OK) st = cuda_check(cudaStreamSynchronize(s), "count read-back");
  if (st != HS_OK) return st;
  for (int h = 0; h < W; ++h) {
    cnt[h] = pairs[2 * h] < 0 ? 0 : pairs[2 * h];
    caps[h] = pairs[2 * h + 1];
  }
  int64_t D = 0;
  for (int h = 0; h < W; ++h) D += cnt[h];
  const int64_t R = n_dest;
  auto lo = [&](int64_t d) { return d * D / R; };
  // send[g][h]: rank g's global slice [off_g, off_g + D_g) intersected with rank h's block
  auto plan = [&](int g, int h) -> int64_t {
    if (is_dest[h] < 0) return 0;
    int64_t off = 0;
    for (int x = 0; x < g; ++x) off += cnt[x];
    const int64_t d = is_dest[h], a = std::max(off, lo(d)), b = std::min(off + cnt[g], lo(d + 1));
    return b > a ? b - a : 0;
  };
  // the same decision on every rank: does any receiver's block exceed its capacity?
  for (int h = 0; h < W; ++h) {
    const int64_t blk = is_dest[h] < 0 ? 0 : lo(is_dest[h] + 1) - lo(is_dest[h]);
    if (blk > caps[h])
      return fail(HS_ERR_INVALID_ARGUMENT, "rank %d: recv_cap %lld < %lld rows to receive (no rank exchanged)",
                  h, (long long)caps[h], (long long)blk);
  }
  std::vector<int64_t> scnt(W), soff(W), rcnt(W), roff(W);
  int64_t so = 0, ro = 0;
  for (int h = 0; h < W; ++h) {
    scnt[h] = plan(rank, h);
    soff[h] = so;
    so += scnt[h];
    rcnt[h] = plan(h, rank);
    roff[h] = ro;
    ro += rcnt[h];
  }
  r = hs::nccl_exchange(reinterpret_cast<const char*>(ids), soff.data(), scnt.data(),
                        reinterpret_cast<char*>(recv_ids), roff.data(), rcnt.data(), 8, comm, s);
  if (r) return fail(HS_ERR_NCCL, "NCCL send/recv (ids): %s", hs::nccl_error(r));
  if (payload_row_bytes) {
    r = hs::nccl_exchange(reinterpret_cast<const char*>(payload), soff.data(), scnt.data(),
                          reinterpret_cast<char*>(recv_payload), roff.data(), rcnt.data(),
                          payload_row_bytes, comm, s);
    if (r) return fail(HS_ERR_NCCL, "NCCL send/recv (payload): %s", hs::nccl_error(r));
  }
  *h_recv_count = ro;
  return HS_OK;
}

size_t hs_route_compact_workspace(int64_t n) { return hs::compact_ws_bytes(n); }

static hs_status_t route_compact_impl(const float* conf, int64_t n, const int64_t* d_n,
                                      float threshold, const float* d_threshold, int32_t is_last, const int64_t* ids,
                                      const int32_t* pred, int32_t pred_len, int64_t* acc_ids,
                                      float* acc_conf, int32_t* acc_pred, int64_t* def_ids,
                                      int64_t* def_pos, const void* payload,
                                      int64_t payload_row_bytes, void* def_payload,
                                      int64_t* d_counts, void* ws, cudaStream_t s) {
  hs::CompactArgs a{};
  a.conf = conf;
  a.n = n;
  a.d_n = d_n;
  a.threshold = threshold;
  a.d_threshold = d_threshold;
  a.is_last = is_last ? 1 : 0;
  a.ids = ids;
  a.pred = pred;
  a.pred_len = pred_len;
  a.acc_ids = acc_ids;
  a.acc_conf = acc_conf;
  a.acc_pred = acc_pred;
  a.def_ids = def_ids;
  a.def_pos = def_pos;
  a.counts = d_counts;
  a.ws = ws;
  hs_status_t st = cuda_check(hs::launch_route_compact(a, s), "route/compact kernel");
  if (st != HS_OK) return st;
  if (def_payload && payload_row_bytes > 0 && !is_last)
    st = cuda_check(hs::launch_gather_rows(def_pos, d_counts + 1, n, payload, payload_row_bytes,
                                           def_payload, s),
                    "gather kernel");
  return st;
}

hs_status_t hs_route_compact(const float* conf, int64_t n, const int64_t* d_n, float threshold,
                             const float* d_threshold, int32_t is_last, const int64_t* ids, const int32_t* pred,
                             int32_t pred_len, int64_t* acc_ids, float* acc_conf,
                             int32_t* acc_pred, int64_t* def_ids, int64_t* def_pos,
                             const void* payload, int64_t payload_row_bytes, void* def_payload,
                             int64_t* d_counts, void* ws, size_t ws_bytes, hs_stream_t stream) {
  if (n < 0 || n >= (int64_t(1) << 30)) return fail(HS_ERR_INVALID_ARGUMENT, "n outside 0..2^30-1");
  if (!is_last && !d_threshold) {
    hs_status_t st = check_threshold(threshold);
    if (st != HS_OK) return st;
  }
  if (!d_counts) return fail(HS_ERR_INVALID_ARGUMENT, "d_counts is required");
  if (n > 0 && !conf) return fail(HS_ERR_INVALID_ARGUMENT, "conf is required");
  if (acc_pred && (!pred || pred_len < 1)) return fail(HS_ERR_INVALID_ARGUMENT, "acc_pred requires pred and pred_len >= 1");
  if (def_payload) {
    if (!payload || payload_row_bytes <= 0 || (payload_row_bytes & 15) || !aligned16(payload) || !aligned16(def_payload))
      return fail(HS_ERR_INVALID_ARGUMENT, "payload rows must be 16-byte aligned multiples of 16 bytes");
    if (!def_pos) return fail(HS_ERR_INVALID_ARGUMENT, "def_payload requires def_pos (gather indices)");
  }
  if (!ws || ws_bytes < hs::compact_ws_bytes(n))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, hs::compact_ws_bytes(n));
  return route_compact_impl(conf, n, d_n, threshold, d_threshold, is_last, ids, pred, pred_len,
                            acc_ids, acc_conf, acc_pred, def_ids, def_pos, payload, payload_row_bytes,
                            def_payload, d_counts, ws, (cudaStream_t)stream);
}

hs_status_t hs_skip_edges(float threshold, int32_t successors, int32_t mode, float* edges) {
  if (successors < 1 || successors - 1 > hs::kMaxSkipEdges)
    return fail(HS_ERR_INVALID_ARGUMENT, "successors = %d outside 1..%d", successors, hs::kMaxSkipEdges + 1);
  if (mode != 0 && mode != 1) return fail(HS_ERR_INVALID_ARGUMENT, "skip mode must be 0 or 1");
  if (successors > 1 && !edges) return fail(HS_ERR_INVALID_ARGUMENT, "edges is NULL");
  double p10 = 1.0;
  for (int i = 1; i < successors; ++i) {
    p10 *= 10.0;
    edges[i - 1] = mode == 1 ? (float)((double)threshold / p10)
                             : (float)((double)threshold * (double)(successors - i) / (double)successors);
  }
  return HS_OK;
}

hs_status_t hs_skip_select(const int32_t* dest, int64_t n_req, int32_t stage, int64_t* batch_ids,
                           int64_t* d_counts, void* ws, size_t ws_bytes, hs_stream_t stream) {
  if (n_req < 0 || n_req >= (int64_t(1) << 30)) return fail(HS_ERR_INVALID_ARGUMENT, "n_req outside 0..2^30-1");
  if (!d_counts || (n_req > 0 && (!dest || !batch_ids))) return fail(HS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (!ws || ws_bytes < hs::compact_ws_bytes(n_req))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, hs::compact_ws_bytes(n_req));
  hs::CompactArgs a{};
  a.n = n_req;
  a.sel_dest = dest;
  a.sel_k = stage;
  a.def_ids = batch_ids;
  a.counts = d_counts;
  a.ws = ws;
  return cuda_check(hs::launch_route_compact(a, (cudaStream_t)stream), "skip select kernel");
}

hs_status_t hs_skip_route(const float* conf, int64_t n, const int64_t* d_n, float threshold,
                          const float* d_threshold, int32_t stage, int32_t n_stages, int32_t mode,
                          const int64_t* ids, const int32_t* pred, int32_t pred_len,
                          int64_t* acc_ids, float* acc_conf, int32_t* acc_pred, int32_t* dest,
                          int64_t* d_counts, void* ws, size_t ws_bytes, hs_stream_t stream) {
  if (n < 0 || n >= (int64_t(1) << 30)) return fail(HS_ERR_INVALID_ARGUMENT, "n outside 0..2^30-1");
  if (n_stages < 1 || n_stages - 2 > hs::kMaxSkipEdges || stage < 0 || stage >= n_stages)
    return fail(HS_ERR_INVALID_ARGUMENT, "stage %d / n_stages %d out of range", stage, n_stages);
  if (mode != 0 && mode != 1) return fail(HS_ERR_INVALID_ARGUMENT, "skip mode must be 0 or 1");
  const int is_last = stage == n_stages - 1;
  if (!is_last && !d_threshold) {
    hs_status_t st = check_threshold(threshold);
    if (st != HS_OK) return st;
  }
  if (!d_counts || (n > 0 && (!conf || !ids || !dest))) return fail(HS_ERR_INVALID_ARGUMENT, "NULL argument");
  if (acc_pred && (!pred || pred_len < 1)) return fail(HS_ERR_INVALID_ARGUMENT, "acc_pred requires pred and pred_len >= 1");
  if (!ws || ws_bytes < hs::compact_ws_bytes(n))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, hs::compact_ws_bytes(n));
  hs::CompactArgs a{};
  a.conf = conf;
  a.n = n;
  a.d_n = d_n;
  a.threshold = threshold;
  a.d_threshold = d_threshold;
  a.is_last = is_last;
  a.ids = ids;
  a.pred = pred;
  a.pred_len = pred_len;
  a.acc_ids = acc_ids;
  a.acc_conf = acc_conf;
  a.acc_pred = acc_pred;
  a.counts = d_counts;
  a.ws = ws;
  a.skip_dest = dest;
  a.skip_K = n_stages;
  a.skip_stage = stage;
  a.skip_mode = mode;
  return cuda_check(hs::launch_route_compact(a, (cudaStream_t)stream), "skip route kernel");
}

// cascade-step workspace: [compact ws][conf f32 n][argmax i32 n*L][def_pos i64 n][conf ws]
static size_t step_layout(int64_t n, int32_t L, size_t* o_conf, size_t* o_am, size_t* o_pos,
                          size_t* o_cws, size_t* o_tick = nullptr, size_t* o_split = nullptr,
                          size_t* o_fuse = nullptr) {
  size_t off = align_up(hs::compact_ws_bytes(n), 256);
  if (o_tick) *o_tick = off;           // K1 row-group ticket + finished-CTA count
  off += 256;
  if (o_fuse) *o_fuse = off;           // fused K1+K3: epoch + two banks of tile counters
  off = align_up(off + hs::fuse_ws_bytes(), 256);
  *o_conf = off;
  off = align_up(off + (size_t)n * sizeof(float), 256);
  *o_am = off;
  off = align_up(off + (size_t)n * (size_t)L * sizeof(int32_t), 256);
  *o_pos = off;
  off = align_up(off + (size_t)n * sizeof(int64_t), 256);
  *o_cws = off;
  off = align_up(off + conf_ws(n, L), 256);
  if (o_split) *o_split = off;         // K1e split-row partials (small batches), zero-filled once
  // the split-row region is reserved for min(n*L, kSplitMaxRows) rows, so the
  // workspace size never shrinks as n grows (a workspace sized for a capacity
  // serves every smaller batch, including those that take the split path)
  const int64_t srows = n * (int64_t)L < hs::kSplitMaxRows ? n * (int64_t)L : hs::kSplitMaxRows;
  off = align_up(off + hs::split_ws_bytes(srows), 256);
  return off;
}

size_t hs_cascade_step_workspace(int64_t n, int32_t seq_len) {
  size_t a, b, c, d;
  return step_layout(n < 0 ? 0 : n, seq_len < 1 ? 1 : seq_len, &a, &b, &c, &d);
}

hs_status_t hs_cascade_step(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                            int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                            const int64_t* row_index, const int64_t* d_n, float temperature,
                            hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                            const float* d_threshold, const int64_t* ids, const void* payload, int64_t payload_row_bytes,
                            int64_t* acc_ids, float* acc_conf, int32_t* acc_pred,
                            int64_t* next_ids, void* next_payload, int64_t* d_counts, void* ws,
                            size_t ws_bytes, uint32_t* d_status, hs_stream_t stream) {
  return hs_cascade_step_ex(stage, n_stages, logits, dtype, n, seq_len, n_classes, row_stride,
                            row_index, d_n, temperature, kind, reduce, threshold, d_threshold, ids,
                            payload, payload_row_bytes, acc_ids, acc_conf, acc_pred, next_ids,
                            next_payload, d_counts, ws, ws_bytes, d_status, 0, 0u, stream);
}

// HS_FUSE=1: hs_cascade_step runs K1 with the threshold test and the stable
// compaction fused into it (one launch per stage).  Opt-in: measured slower
// than K1 then K3 on C2.
static bool fuse_enabled() {
  const char* e = getenv("HS_FUSE");
  return e && e[0] == '1';
}

static hs_status_t step_common_checks(int32_t stage, int32_t n_stages, int64_t n, float threshold,
                                      const float* d_threshold, int32_t top_k) {
  if (top_k < 0 || top_k > hs::kTopkMax)
    return fail(HS_ERR_INVALID_ARGUMENT, "top_k = %d outside 0..%d", top_k, hs::kTopkMax);
  if (n_stages < 1 || stage < 0 || stage >= n_stages)
    return fail(HS_ERR_INVALID_ARGUMENT, "stage %d outside 0..n_stages-1 (%d)", stage, n_stages);
  if (n < 0 || n >= (int64_t(1) << 30)) return fail(HS_ERR_INVALID_ARGUMENT, "n must be in 0..2^30-1 per call");
  if (stage != n_stages - 1 && !d_threshold) return check_threshold(threshold);
  return HS_OK;
}

// The last stage's step without a compaction (HS_LAST_K3=1 restores it): it
// accepts every row in order, so K1 writes the accepted lists itself.
static bool last_direct_enabled() {
  const char* e = getenv("HS_LAST_K3");
  return !(e && e[0] == '1');
}

struct LastOut {                    // the last stage written by K1 (NULL: K1's own buffers)
  float* conf;
  int32_t* pred;
  const int64_t* ids;
  int64_t* ids_out;
  int64_t* counts;
};

static hs_status_t cascade_confidence_impl(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                                           int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                                           const int64_t* row_index, const int64_t* d_n, float temperature,
                                           hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                                           const float* d_threshold, uint64_t* d_defer_count, void* ws,
                                           size_t ws_bytes, uint32_t* d_status, int32_t top_k, uint32_t flags,
                                           hs_stream_t stream, const LastOut* last);

hs_status_t hs_cascade_confidence(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                                  int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                                  const int64_t* row_index, const int64_t* d_n, float temperature,
                                  hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                                  const float* d_threshold, uint64_t* d_defer_count, void* ws,
                                  size_t ws_bytes, uint32_t* d_status, int32_t top_k, uint32_t flags,
                                  hs_stream_t stream) {
  return cascade_confidence_impl(stage, n_stages, logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n,
                                 temperature, kind, reduce, threshold, d_threshold, d_defer_count, ws, ws_bytes,
                                 d_status, top_k, flags, stream, nullptr);
}

static hs_status_t cascade_confidence_impl(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                                           int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                                           const int64_t* row_index, const int64_t* d_n, float temperature,
                                           hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                                           const float* d_threshold, uint64_t* d_defer_count, void* ws,
                                           size_t ws_bytes, uint32_t* d_status, int32_t top_k, uint32_t flags,
                                           hs_stream_t stream, const LastOut* last) {
  if (flags & ~(uint32_t)(HS_STEP_OVERLAP_PREVIOUS | HS_STEP_LOGITS_CAPACITY))
    return fail(HS_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  hs_status_t st = step_common_checks(stage, n_stages, n, threshold, d_threshold, top_k);
  if (st != HS_OK) return st;
  st = check_logits(logits, dtype, n, seq_len, n_classes, row_stride, temperature, kind, reduce);
  if (st != HS_OK) return st;
  size_t o_conf, o_am, o_pos, o_cws, o_tick, o_split;
  const size_t need = step_layout(n, seq_len, &o_conf, &o_am, &o_pos, &o_cws, &o_tick, &o_split);
  if (!ws || ws_bytes < need) return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
  if (n == 0) return HS_OK;
  cudaStream_t s = (cudaStream_t)stream;
  char* w = reinterpret_cast<char*>(ws);
  float* conf = reinterpret_cast<float*>(w + o_conf);
  int32_t* am = reinterpret_cast<int32_t*>(w + o_am);
  hs::ConfArgs a = make_conf_args(logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n,
                                  temperature, kind);
  a.top_k = top_k;
  if (hs::split_ws_bytes(n * (int64_t)seq_len)) a.split_ws = w + o_split;
  if (flags & HS_STEP_OVERLAP_PREVIOUS) {
    // CTAs that start late (SMs held by the previous kernel) take fewer rows
    a.ticket = reinterpret_cast<unsigned int*>(w + o_tick);
    a.late_wait = 1;
  }
  a.rows_cap_valid = (flags & HS_STEP_LOGITS_CAPACITY) ? 1 : 0;
  if (last) {
    if (last->conf) conf = last->conf;
    if (last->pred) am = last->pred;
    a.last_ids = last->ids;
    a.last_ids_out = last->ids_out;
    a.last_counts = last->counts;
  }
  st = run_confidence_args(a, dtype, reduce, conf, am, nullptr, nullptr, w + o_cws, d_status, s);
  if (st != HS_OK || !d_defer_count) return st;
  return cuda_check(hs::launch_count_deferred(conf, n, d_n, threshold, d_threshold, stage == n_stages - 1,
                                              reinterpret_cast<unsigned long long*>(d_defer_count), s),
                    "count kernel");
}

hs_status_t hs_cascade_compact(int32_t stage, int32_t n_stages, int64_t n, int32_t seq_len,
                               const int64_t* d_n, float threshold, const float* d_threshold,
                               const int64_t* ids, const void* payload, int64_t payload_row_bytes,
                               int64_t* acc_ids, float* acc_conf, int32_t* acc_pred, int64_t* next_ids,
                               void* next_payload, int64_t* d_counts, void* ws, size_t ws_bytes,
                               hs_stream_t stream) {
  hs_status_t st = step_common_checks(stage, n_stages, n, threshold, d_threshold, 0);
  if (st != HS_OK) return st;
  if (seq_len < 1) return fail(HS_ERR_INVALID_ARGUMENT, "seq_len = %d < 1", seq_len);
  if (!d_counts) return fail(HS_ERR_INVALID_ARGUMENT, "d_counts is required");
  if (next_payload && (!payload || payload_row_bytes <= 0 || (payload_row_bytes & 15) ||
                       !aligned16(payload) || !aligned16(next_payload)))
    return fail(HS_ERR_INVALID_ARGUMENT, "payload rows must be 16-byte aligned multiples of 16 bytes");
  size_t o_conf, o_am, o_pos, o_cws, o_tick, o_split;
  const size_t need = step_layout(n, seq_len, &o_conf, &o_am, &o_pos, &o_cws, &o_tick, &o_split);
  if (!ws || ws_bytes < need) return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = (cudaStream_t)stream;
  if (n == 0) return cuda_check(cudaMemsetAsync(d_counts, 0, 2 * sizeof(int64_t), s), "memset counts");
  char* w = reinterpret_cast<char*>(ws);
  const float* conf = reinterpret_cast<const float*>(w + o_conf);
  const int32_t* am = reinterpret_cast<const int32_t*>(w + o_am);
  int64_t* pos = reinterpret_cast<int64_t*>(w + o_pos);
  return route_compact_impl(conf, n, d_n, threshold, d_threshold, stage == n_stages - 1, ids, am, seq_len,
                            acc_ids, acc_conf, acc_pred, next_ids, next_payload ? pos : nullptr, payload,
                            payload_row_bytes, next_payload, d_counts, ws, s);
}

hs_status_t hs_cascade_step_ex(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                               int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                               const int64_t* row_index, const int64_t* d_n, float temperature,
                               hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                               const float* d_threshold, const int64_t* ids, const void* payload,
                               int64_t payload_row_bytes, int64_t* acc_ids, float* acc_conf,
                               int32_t* acc_pred, int64_t* next_ids, void* next_payload,
                               int64_t* d_counts, void* ws, size_t ws_bytes, uint32_t* d_status,
                               int32_t top_k, uint32_t flags, hs_stream_t stream) {
  // validate both halves before launching either
  if (flags & ~(uint32_t)(HS_STEP_OVERLAP_PREVIOUS | HS_STEP_LOGITS_CAPACITY))
    return fail(HS_ERR_INVALID_ARGUMENT, "unknown flags 0x%x", flags);
  hs_status_t st = step_common_checks(stage, n_stages, n, threshold, d_threshold, top_k);
  if (st != HS_OK) return st;
  if (!d_counts) return fail(HS_ERR_INVALID_ARGUMENT, "d_counts is required");
  if (next_payload && (!payload || payload_row_bytes <= 0 || (payload_row_bytes & 15) ||
                       !aligned16(payload) || !aligned16(next_payload)))
    return fail(HS_ERR_INVALID_ARGUMENT, "payload rows must be 16-byte aligned multiples of 16 bytes");
  // the last stage accepts every row in order: K1 writes the accepted lists
  // and the counts itself (one launch, no compaction)
  if (stage == n_stages - 1 && seq_len == 1 && last_direct_enabled()) {
    if (n == 0) return cuda_check(cudaMemsetAsync(d_counts, 0, 2 * sizeof(int64_t), (cudaStream_t)stream),
                                  "memset counts");
    const LastOut last{acc_conf, acc_pred, ids, acc_ids, d_counts};
    return cascade_confidence_impl(stage, n_stages, logits, dtype, n, seq_len, n_classes, row_stride, row_index,
                                   d_n, temperature, kind, reduce, threshold, d_threshold, nullptr, ws, ws_bytes,
                                   d_status, top_k, flags, stream, &last);
  }
  // HS_FUSE=1: one launch, K1 with the threshold test and the stable
  // compaction in its row epilogue, when the rows take the cp.async kernel
  if (!(flags & HS_STEP_OVERLAP_PREVIOUS) && fuse_enabled()) {
    st = check_logits(logits, dtype, n, seq_len, n_classes, row_stride, temperature, kind, reduce);
    if (st != HS_OK) return st;
    size_t o_conf, o_am, o_pos, o_cws, o_tick, o_split, o_fuse;
    const size_t need = step_layout(n, seq_len, &o_conf, &o_am, &o_pos, &o_cws, &o_tick, &o_split, &o_fuse);
    if (!ws || ws_bytes < need) return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, need);
    char* w = reinterpret_cast<char*>(ws);
    hs::ConfArgs a = make_conf_args(logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n,
                                    temperature, kind);
    a.top_k = top_k;
    a.rows_cap_valid = (flags & HS_STEP_LOGITS_CAPACITY) ? 1 : 0;
    if (hs::confidence_fusable(a)) {
      cudaStream_t s = (cudaStream_t)stream;
      if (n == 0) return cuda_check(cudaMemsetAsync(d_counts, 0, 2 * sizeof(int64_t), s), "memset counts");
      const int is_last = stage == n_stages - 1;
      int64_t* pos = reinterpret_cast<int64_t*>(w + o_pos);
      a.fz.on = 1;
      a.fz.is_last = is_last;
      a.fz.threshold = threshold;
      a.fz.d_threshold = d_threshold;
      a.fz.ids = ids;
      a.fz.acc_ids = acc_ids;
      a.fz.acc_conf = acc_conf;
      a.fz.acc_pred = acc_pred;
      a.fz.def_ids = next_ids;
      a.fz.def_pos = (next_payload && !is_last) ? pos : nullptr;
      a.fz.counts = d_counts;
      a.fz.tiles = w + o_fuse;
      st = run_confidence_args(a, dtype, reduce, reinterpret_cast<float*>(w + o_conf),
                               reinterpret_cast<int32_t*>(w + o_am), nullptr, nullptr, w + o_cws, d_status, s);
      if (st != HS_OK) return st;
      if (next_payload && payload_row_bytes > 0 && !is_last)
        st = cuda_check(hs::launch_gather_rows(pos, d_counts + 1, n, payload, payload_row_bytes, next_payload, s),
                        "gather kernel");
      return st;
    }
  }
  st = hs_cascade_confidence(stage, n_stages, logits, dtype, n, seq_len, n_classes, row_stride, row_index, d_n,
                             temperature, kind, reduce, threshold, d_threshold, nullptr, ws, ws_bytes, d_status,
                             top_k, flags, stream);
  if (st != HS_OK) return st;
  return hs_cascade_compact(stage, n_stages, n, seq_len, d_n, threshold, d_threshold, ids, payload,
                            payload_row_bytes, acc_ids, acc_conf, acc_pred, next_ids, next_payload, d_counts,
                            ws, ws_bytes, stream);
}

size_t hs_calibrate_workspace(int32_t K, int32_t log2_bins) {
  if (log2_bins < 1 || log2_bins > 14) return 0;
  return hs::calib_ws_bytes(K, log2_bins);
}
size_t hs_calibrate_hist_bytes(int32_t log2_bins) {
  if (log2_bins < 1 || log2_bins > 14) return 0;
  return hs::calib_hist_bytes(log2_bins);
}
int32_t* hs_calibrate_hist_ptr(void* ws) {
  return reinterpret_cast<int32_t*>(reinterpret_cast<char*>(ws) + sizeof(hs::CalibState));
}

static hs_status_t check_calib(int32_t K, int32_t q, void* ws, size_t ws_bytes) {
  if (K < 2 || K > 17) return fail(HS_ERR_INVALID_ARGUMENT, "K = %d outside 2..17", K);
  if (q < 1 || q > 14) return fail(HS_ERR_INVALID_ARGUMENT, "log2_bins = %d outside 1..14", q);
  if (!ws || ws_bytes < hs::calib_ws_bytes(K, q))
    return fail(HS_ERR_WORKSPACE_TOO_SMALL, "workspace %zu < %zu", ws_bytes, hs::calib_ws_bytes(K, q));
  return HS_OK;
}

hs_status_t hs_calibrate_begin(int32_t K, int32_t log2_bins, int64_t target_correct, void* ws,
                               size_t ws_bytes, hs_stream_t stream) {
  hs_status_t st = check_calib(K, log2_bins, ws, ws_bytes);
  if (st != HS_OK) return st;
  return cuda_check(hs::launch_calib_init(ws, log2_bins, target_correct, (cudaStream_t)stream), "calib init");
}

hs_status_t hs_calibrate_histogram(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                   int32_t log2_bins, int32_t round, const int32_t* d_bin_idx,
                                   void* ws, size_t ws_bytes, hs_stream_t stream) {
  hs_status_t st = check_calib(K, log2_bins, ws, ws_bytes);
  if (st != HS_OK) return st;
  if (N < 0) return fail(HS_ERR_INVALID_ARGUMENT, "N < 0");
  if (round < 0 || round > K - 2) return fail(HS_ERR_INVALID_ARGUMENT, "round outside 0..K-2");
  if (N == 0) return HS_OK;   // an empty shard contributes nothing
  if (!conf || !correct || (round > 0 && !d_bin_idx)) return fail(HS_ERR_INVALID_ARGUMENT, "NULL input");
  return cuda_check(hs::launch_calib_hist(conf, correct, K, N, log2_bins, round, d_bin_idx,
                                          hs_calibrate_hist_ptr(ws), (cudaStream_t)stream),
                    "calib histogram");
}

hs_status_t hs_calibrate_select(int32_t K, int32_t log2_bins, int32_t round, int32_t* d_bin_idx,
                                float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                int64_t* d_correct_total, void* ws, size_t ws_bytes,
                                hs_stream_t stream) {
  hs_status_t st = check_calib(K, log2_bins, ws, ws_bytes);
  if (st != HS_OK) return st;
  if (round < 0 || round > K - 2) return fail(HS_ERR_INVALID_ARGUMENT, "round outside 0..K-2");
  if (!d_bin_idx || !d_thresholds || !d_reach || !d_handled || !d_correct_total)
    return fail(HS_ERR_INVALID_ARGUMENT, "NULL output");
  return cuda_check(hs::launch_calib_select(K, log2_bins, round, d_bin_idx, d_thresholds, d_reach,
                                            d_handled, d_correct_total, ws, (cudaStream_t)stream),
                    "calib select");
}

static hs_status_t calibrate_greedy(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                    int32_t log2_bins, int64_t target_correct, int32_t* d_bin_idx,
                                    float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                    int64_t* d_correct_total, void* ws, size_t ws_bytes,
                                    hs_stream_t stream) {
  hs_status_t st = HS_OK;
  // default: all rounds in one cooperative launch; HS_CALIB_MODE=cluster|split
  // selects the one-cluster (DSMEM) kernel or per-round launches (tests / A-B)
  const char* mode = getenv("HS_CALIB_MODE");
  if (mode && !strcmp(mode, "cluster") && N < (1 << 20))
    return cuda_check(hs::launch_calib_cluster(conf, correct, K, N, log2_bins, target_correct,
                                               d_bin_idx, d_thresholds, d_reach, d_handled,
                                               d_correct_total, ws, (cudaStream_t)stream),
                      "calib cluster kernel");
  if (!mode || strcmp(mode, "split"))
    return cuda_check(hs::launch_calib_fused(conf, correct, K, N, log2_bins, target_correct,
                                             d_bin_idx, d_thresholds, d_reach, d_handled,
                                             d_correct_total, ws, (cudaStream_t)stream),
                      "calib fused (cooperative) kernel");
  st = hs_calibrate_begin(K, log2_bins, target_correct, ws, ws_bytes, stream);
  for (int k = 0; st == HS_OK && k < K - 1; ++k) {
    st = hs_calibrate_histogram(conf, correct, K, N, log2_bins, k, d_bin_idx, ws, ws_bytes, stream);
    if (st == HS_OK)
      st = hs_calibrate_select(K, log2_bins, k, d_bin_idx, d_thresholds, d_reach, d_handled,
                               d_correct_total, ws, ws_bytes, stream);
  }
  return st;
}

hs_status_t hs_calibrate_thresholds(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                    int32_t log2_bins, int64_t target_correct,
                                    int32_t refine_passes, int32_t* d_bin_idx,
                                    float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                    int64_t* d_correct_total, void* ws, size_t ws_bytes,
                                    hs_stream_t stream) {
  hs_status_t st = check_calib(K, log2_bins, ws, ws_bytes);
  if (st != HS_OK) return st;
  if (N <= 0) return fail(HS_ERR_INVALID_ARGUMENT, "empty validation set (N = %lld)", (long long)N);
  if (refine_passes < 0 || refine_passes > 64)
    return fail(HS_ERR_INVALID_ARGUMENT, "refine_passes = %d outside 0..64", refine_passes);
  if (!conf || !correct) return fail(HS_ERR_INVALID_ARGUMENT, "NULL input");
  if (!d_bin_idx || !d_thresholds || !d_reach || !d_handled || !d_correct_total)
    return fail(HS_ERR_INVALID_ARGUMENT, "NULL output");
  st = calibrate_greedy(conf, correct, K, N, log2_bins, target_correct, d_bin_idx, d_thresholds,
                        d_reach, d_handled, d_correct_total, ws, ws_bytes, stream);
  if (st != HS_OK || refine_passes == 0) return st;
  return cuda_check(hs::launch_calib_refine(conf, correct, K, N, log2_bins, refine_passes, d_bin_idx,
                                            d_thresholds, d_reach, d_handled, d_correct_total, ws,
                                            (cudaStream_t)stream),
                    "calib refinement");
}

hs_status_t hs_calibrate_thresholds_peer(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                         int32_t log2_bins, int64_t target_correct, int32_t* d_bin_idx,
                                         float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                         int64_t* d_correct_total, const hs_peer_t* g, void* ws,
                                         size_t ws_bytes, uint32_t* d_status, hs_stream_t stream) {
  hs_status_t st = check_calib(K, log2_bins, ws, ws_bytes);
  if (st != HS_OK) return st;
  hs::PeerArgs A;
  hs::PeerLayout L;
  st = peer_args(g, false, &A, &L);
  if (st != HS_OK) return st;
  if (g->log2_bins != log2_bins)
    return fail(HS_ERR_INVALID_ARGUMENT, "the group's regions were sized for log2_bins = %d", g->log2_bins);
  if (N < 0 || (N > 0 && (!conf || !correct))) return fail(HS_ERR_INVALID_ARGUMENT, "N >= 0 and inputs required");
  if (K > 16) return fail(HS_ERR_UNSUPPORTED, "K = %d > 16 on the peer path", K);
  if (N * (int64_t)g->world >= ((int64_t)1 << 21))
    return fail(HS_ERR_UNSUPPORTED, "N * world must be < 2^21 on the peer path (packed bins)");
  if (!d_bin_idx || !d_thresholds || !d_reach || !d_handled || !d_correct_total)
    return fail(HS_ERR_INVALID_ARGUMENT, "NULL output");
  hs::PeerCal pc{};
  pc.world = g->world;
  pc.rank = g->rank;
  for (int h = 0; h < g->world; ++h) {
    pc.slots[h] = reinterpret_cast<unsigned long long*>(reinterpret_cast<char*>(g->region[h]) + L.cal_off);
    pc.arrive[h] = A.hdr[h]->cal_arrive;
  }
  pc.round_ctr = &A.hdr[g->rank]->cal_round;
  pc.status = d_status;
  const cudaError_t e = hs::launch_calib_peer(conf, correct, K, N, log2_bins, target_correct, d_bin_idx,
                                              d_thresholds, d_reach, d_handled, d_correct_total, ws, pc,
                                              (cudaStream_t)stream);
  if (e == cudaErrorNotSupported)
    return fail(HS_ERR_UNSUPPORTED, "the shard does not fit the resident calibration kernel");
  return cuda_check(e, "peer calibration kernel");
}

hs_status_t hs_cascade_step_peer(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                                 int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                                 const int64_t* row_index, const int64_t* d_n, float temperature,
                                 hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                                 const float* d_threshold, const int64_t* ids, const void* payload,
                                 int64_t payload_row_bytes, int64_t* acc_ids, float* acc_conf,
                                 int32_t* acc_pred, int64_t* next_ids, void* next_payload,
                                 int64_t* d_counts, void* ws, size_t ws_bytes, uint32_t* d_status,
                                 int32_t top_k, uint32_t flags, const hs_peer_t* g, int32_t set,
                                 const int32_t* next_stage_ranks, int32_t n_next_ranks,
                                 int64_t* d_recv_count, hs_stream_t stream) {
  const int is_last = stage == n_stages - 1;
  if (!is_last) {     // validate the forward before anything is launched
    hs::PeerArgs A;
    hs_status_t st = peer_args(g, next_payload != nullptr, &A, nullptr);
    if (st != HS_OK) return st;
    hs::PeerDest d{};
    st = peer_dest(g, next_stage_ranks, n_next_ranks, &d);
    if (st != HS_OK) return st;
    if (set < 0 || set > 1 || !next_ids || !d_recv_count)
      return fail(HS_ERR_INVALID_ARGUMENT, "set in {0,1}, next_ids and d_recv_count are required");
    if (n > g->cap) return fail(HS_ERR_INVALID_ARGUMENT, "n = %lld exceeds the group's cap", (long long)n);
  }
  hs_status_t st = hs_cascade_step_ex(stage, n_stages, logits, dtype, n, seq_len, n_classes, row_stride,
                                      row_index, d_n, temperature, kind, reduce, threshold, d_threshold, ids,
                                      payload, payload_row_bytes, acc_ids, acc_conf, acc_pred, next_ids,
                                      next_payload, d_counts, ws, ws_bytes, d_status, top_k, flags, stream);
  if (st != HS_OK || is_last) return st;
  return hs_peer_forward(g, set, next_ids, next_payload, d_counts + 1, next_stage_ranks, n_next_ranks,
                         d_recv_count, d_status, stream);
}

}  // extern "C"
