/*
 * include/hs.h -- C-ABI of libhs.so, the B200 (sm_100a) HybridServe cascade router.
 *
 * The library implements the data-parallel hot path of HybridServe (arXiv
 * 2505.12566): per-request confidence from a stage model's logits, the
 * threshold test, stable compaction + gather of the deferred requests into the
 * next stage's batch, and offline Accuracy-Preserving threshold calibration.
 * Citations "P:<n>" are line numbers of the paper's text; the
 * readings taken where the paper is garbled are listed in DESIGN.md.
 *
 * Conventions (all entry points):
 *  - Pointers are DEVICE pointers unless marked "host".  The caller owns every
 *    buffer; the library never allocates device memory and never synchronises
 *    the device or the stream.  Every data call is asynchronous and ordered on
 *    the given CUDA stream; passing 0 selects the legacy default stream.
 *  - Argument errors are detected on the host before any launch and leave all
 *    outputs untouched (HS_ERR_INVALID_ARGUMENT).  hs_last_error() returns a
 *    thread-local detail string for the most recent failure.
 *  - Data errors (a NaN or +inf logit, or a row whose entries are all -inf;
 *    the paper's prediction vectors are finite probabilities) cannot be
 *    known at return time: the kernel ORs bit 0 (HS_STATUS_NONFINITE) into
 *    *d_status (optional device word) and writes conf = NaN, argmax = -1 for
 *    that row.  A NaN confidence is deferred at every stage but the last.
 *    -inf is accepted as a masked class (probability 0).
 *  - Counts that size later work may live on the device ("d_n" arguments):
 *    when non-NULL, the kernels read the actual item count from *d_n (which
 *    must be <= the host capacity argument).  This lets a whole K-stage
 *    cascade run without a host round trip and be captured in a CUDA graph.
 *  - Alignment: logits base and row_stride * element size must be multiples of
 *    16 bytes (128-bit vector loads); payload rows likewise.
 *  - Determinism: outputs are bitwise identical run to run (fixed reduction
 *    trees, integer histograms, stable compaction).
 *  - Reentrancy: calls are reentrant; a workspace must not be shared by two
 *    calls that may be in flight at the same time.
 */
#ifndef HS_H_
#define HS_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct CUstream_st* hs_stream_t; /* == cudaStream_t */

typedef enum {
  HS_OK = 0,
  HS_ERR_INVALID_ARGUMENT = 1,
  HS_ERR_NONFINITE_INPUT = 2, /* reserved for host-side checks of d_status */
  HS_ERR_CUDA = 3,
  HS_ERR_NCCL = 4,            /* an NCCL call of the hs_comm_* paths failed (hs_last_error: detail) */
  HS_ERR_WORKSPACE_TOO_SMALL = 5,
  HS_ERR_UNSUPPORTED = 6
} hs_status_t;

typedef enum { HS_F32 = 0, HS_BF16 = 1 } hs_dtype_t;

/* Confidence score f_theta(P) of one prediction vector, z = x / T (Temperature
 * Scaling; Eq. 1 P:384-389 fits T offline):
 *   MAXPROB    c = max_j softmax(z)_j             (north_star; reading G1 of P:415)
 *   MAXPROB_SQ c = (max_j softmax(z)_j)^2         ("max(theta(P)^2)" taken literally)
 *   ENTROPY    c = exp(-H), H = -sum_j p_j ln p_j (north_star; 1/perplexity, reading G3) */
typedef enum { HS_CONF_MAXPROB = 0, HS_CONF_MAXPROB_SQ = 1, HS_CONF_ENTROPY = 2 } hs_conf_kind_t;

/* Token -> sequence reduction for generation models ("the minimal
 * confidence is the confidence of complete output"); QA is MIN with L = 2
 * (P:427-430).  NONE requires seq_len == 1. */
typedef enum { HS_SEQ_NONE = 0, HS_SEQ_MIN = 1, HS_SEQ_MEAN = 2 } hs_seq_reduce_t;

#define HS_STATUS_NONFINITE 1u
#define HS_STATUS_NOT_CONVERGED 2u   /* hs_fit_temperature: pass budget exhausted */
#define HS_STATUS_TIMEOUT 4u         /* hs_peer_* / *_peer: a peer did not publish within 10 s */
#define HS_STATUS_OVERFLOW 8u        /* hs_peer_forward*: a rank deferred more than the group's cap */

/* ------------------------------------------------------------------------ */
/* Confidence.                                        */
/* ------------------------------------------------------------------------ */
/* Batch item i (0 <= i < n) reads sequence r = row_index ? row_index[i] : i;
 * its token t (0 <= t < seq_len) is the logits row r*seq_len + t, starting at
 * element (r*seq_len + t) * row_stride of `logits` ([rows x row_stride],
 * row-major, dtype elements, n_classes >= 2 valid entries per row).
 * Outputs (per batch item):
 *   conf[i]                    fp32 confidence (sequence-reduced when seq_len > 1)
 *   argmax[i*seq_len + t]      int32 predicted class per token, lowest index on
 *                              ties (optional, may be NULL)
 *   correct[i]                 1 iff argmax == labels[r*seq_len + t] for all t
 *                              (optional; requires labels, int32 indexed like
 *                              the logits rows)
 * Workspace: hs_confidence_workspace(n, seq_len) bytes.  Only the token-row
 * part (n*seq_len*5 bytes, rounded; 0 when seq_len == 1) is required; a
 * workspace of the full size (no zero fill needed) also lets batches of <= 2,048
 * rows of >= 32 KB use the split-row path (K1e: a row cut over many warps),
 * e.g. one Llama-vocabulary vector in ~15 us instead of ~100 us.
 * temperature: > 0 and finite.  Errors: INVALID_ARGUMENT (n_classes < 2,
 * seq_len < 1, NONE with seq_len > 1, bad T, stride < n_classes, misaligned),
 * WORKSPACE_TOO_SMALL, CUDA (launch failure). */
size_t hs_confidence_workspace(int64_t n, int32_t seq_len);
hs_status_t hs_confidence(const void* logits, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                          int64_t n_classes, int64_t row_stride, const int64_t* row_index,
                          const int64_t* d_n, float temperature, hs_conf_kind_t kind,
                          hs_seq_reduce_t reduce, float* conf, int32_t* argmax,
                          const int32_t* labels, uint8_t* correct, void* ws, size_t ws_bytes,
                          uint32_t* d_status, hs_stream_t stream);

/* hs_confidence_topk (NEXT-2; "P = TopK(P)", reading G4): as
 * hs_confidence, with every token row's softmax restricted to its top_k
 * largest logits (0 = the full row, as hs_confidence; top_k >= n_classes is
 * the full row too).  c = p_max / p_max^2 / exp(-H) of the restricted
 * distribution; validity, argmax and correct bits are those of the full row.
 * The K largest VALUES form a unique multiset, so ties at the K-th place do not
 * matter.  top_k outside 0..32 -> INVALID_ARGUMENT. */
hs_status_t hs_confidence_topk(const void* logits, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                               int64_t n_classes, int64_t row_stride, const int64_t* row_index,
                               const int64_t* d_n, float temperature, hs_conf_kind_t kind,
                               hs_seq_reduce_t reduce, int32_t top_k, float* conf, int32_t* argmax,
                               const int32_t* labels, uint8_t* correct, void* ws, size_t ws_bytes,
                               uint32_t* d_status, hs_stream_t stream);

/* hs_confidence_ex: hs_confidence_topk plus conf_entropy (optional, [n]
 * fp32): exp(-H) of every row written alongside conf in the same pass
 * (north_star "max-probability (and entropy) confidence"; reading G3), e.g.
 * MAXPROB in conf and the entropy confidence in conf_entropy.  NaN for an
 * invalid row.  Requires seq_len == 1 (INVALID_ARGUMENT otherwise). */
hs_status_t hs_confidence_ex(const void* logits, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                             int64_t n_classes, int64_t row_stride, const int64_t* row_index,
                             const int64_t* d_n, float temperature, hs_conf_kind_t kind,
                             hs_seq_reduce_t reduce, int32_t top_k, float* conf, float* conf_entropy,
                             int32_t* argmax, const int32_t* labels, uint8_t* correct, void* ws,
                             size_t ws_bytes, uint32_t* d_status, hs_stream_t stream);

/* Every stage model's confidence on the SAME item set in one launch (the
 * calibration input of Alg. 1: "Compute a on D_v" for every model m_1..m_K,
 * P:458-464).  Batch b (0 <= b < n_batches <= 8) reads logits[b] (host array
 * of device pointers, identical shape/stride/dtype) at temperatures[b] (host
 * array); its items are output rows b*n .. b*n + n-1 of conf / correct (and
 * b*n*seq_len.. of argmax).  labels (optional, [n*seq_len], indexed like the
 * logits rows of one batch) are shared by every batch; row_index likewise.
 * Workspace: hs_confidence_batched_workspace(n_batches, n, seq_len). */
size_t hs_confidence_batched_workspace(int32_t n_batches, int64_t n, int32_t seq_len);
hs_status_t hs_confidence_batched(const void* const* logits, const float* temperatures,
                                  int32_t n_batches, hs_dtype_t dtype, int64_t n, int32_t seq_len,
                                  int64_t n_classes, int64_t row_stride,
                                  const int64_t* row_index, hs_conf_kind_t kind,
                                  hs_seq_reduce_t reduce, float* conf, int32_t* argmax,
                                  const int32_t* labels, uint8_t* correct, void* ws,
                                  size_t ws_bytes, uint32_t* d_status, hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Threshold test + stable compaction + gather.       */
/* ------------------------------------------------------------------------ */
/* Item i (0 <= i < n, or *d_n) is ACCEPTED iff is_last || conf[i] >= threshold
 * ("requests with scores below a threshold ... are passed to larger models",
 * P:444; ties accept; the last model answers everything, t_K = 0, Table III),
 * otherwise DEFERRED.  threshold must be in [0,1] or +inf ("defer all").
 * Both lists are stable (increasing i):
 *   acc_ids[j]   = ids ? ids[i] : i        for the j-th accepted item (optional)
 *   acc_conf[j]  = conf[i]                                             (optional)
 *   acc_pred[j*pred_len + t] = pred[i*pred_len + t]                    (optional)
 *   def_ids[j]   = ids ? ids[i] : i        for the j-th deferred item  (optional)
 *   def_pos[j]   = i                                                   (optional)
 *   def_payload[j*P .. +P) = payload[i*P .. +P)   P = payload_row_bytes (optional, P % 16 == 0)
 *   d_counts[0] = #accepted, d_counts[1] = #deferred  (int64, required)
 * d_threshold (optional device float) overrides `threshold` when non-NULL, so
 * thresholds calibrated on the device need no host round trip (its value is
 * not range-checked; a NaN threshold defers everything).
 * Output buffers must hold n entries (worst case); n < 2^30.  Workspace:
 * hs_route_compact_workspace(n) bytes, ZERO-FILLED before its first use and
 * then reused as is: it holds epoch-tagged decoupled look-back descriptors, so
 * no call needs a memset (CUDA-graph friendly). */
size_t hs_route_compact_workspace(int64_t n);
hs_status_t hs_route_compact(const float* conf, int64_t n, const int64_t* d_n, float threshold,
                             const float* d_threshold, int32_t is_last, const int64_t* ids, const int32_t* pred,
                             int32_t pred_len, int64_t* acc_ids, float* acc_conf,
                             int32_t* acc_pred, int64_t* def_ids, int64_t* def_pos,
                             const void* payload, int64_t payload_row_bytes, void* def_payload,
                             int64_t* d_counts, void* ws, size_t ws_bytes, hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Skip connections (NEXT-1; §IV-C, Alg. 2 line 5 P:530).   */
/* ------------------------------------------------------------------------ */
/* A deferred request jumps over models that are unlikely to be confident:
 * stage k (0-based, n_stages = K models) has s = K-1-k successors and s-1
 * band edges inside [0, t_k), each rounded to fp32:
 *   mode 0 uniform ("uniformly partitioned"): e_i = t_k * (s - i) / s
 *   mode 1 decade  ("LogUniform(0, t_i)", P:530 read as S:320):  e_i = t_k / 10^i
 * A request with c < t_k goes to model k + 1 + #{i : c < e_i} (the lowest
 * confidence reaches the largest model).  Requests are tracked in a
 * per-request int32 array dest[n_req] (caller-owned, device): dest[r] = the
 * model r must visit next, or K + k once model k answered it.  Start with
 * dest = 0 for every request.
 *   hs_skip_select: batch of model k = requests r with dest[r] == k, in
 *     increasing r (stable compaction; d_counts = {#other, #selected}).
 *   hs_skip_route: threshold test of a batch (conf[i] of request ids[i]);
 *     accepted -> acc lists exactly as hs_route_compact; every item updates
 *     dest[ids[i]].  d_threshold as in hs_route_compact.
 * Workspaces: hs_route_compact_workspace(n), zero-filled before first use.
 * hs_skip_edges (host-only, pure): the fp32 edges for a host threshold. */
hs_status_t hs_skip_edges(float threshold, int32_t successors, int32_t mode, float* edges /*host [successors-1]*/);
hs_status_t hs_skip_select(const int32_t* dest, int64_t n_req, int32_t stage, int64_t* batch_ids,
                           int64_t* d_counts, void* ws, size_t ws_bytes, hs_stream_t stream);
hs_status_t hs_skip_route(const float* conf, int64_t n, const int64_t* d_n, float threshold,
                          const float* d_threshold, int32_t stage, int32_t n_stages, int32_t mode,
                          const int64_t* ids, const int32_t* pred, int32_t pred_len,
                          int64_t* acc_ids, float* acc_conf, int32_t* acc_pred, int32_t* dest,
                          int64_t* d_counts, void* ws, size_t ws_bytes, hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* One cascade stage m_k: confidence -> threshold test -> compaction/gather.  */
/* ------------------------------------------------------------------------ */
/* stage: 0-based index k of the model; is_last = (stage == n_stages - 1).
 * The batch is items 0..n-1 (or *d_n); item i has request id ids[i] (NULL =
 * identity) and reads its logits via row_index (NULL = dense, row i; pass
 * row_index == ids when the stage's logits are indexed by request id).
 * Accepted items go to acc_ids / acc_conf / acc_pred (pred = the seq_len
 * argmaxes); deferred items become the next stage's batch: next_ids,
 * next_payload (optional).  d_counts = {#accepted, #deferred}.  d_threshold as
 * for hs_route_compact.
 * Workspace: hs_cascade_step_workspace(n, seq_len) bytes (non-decreasing in n: a
 * workspace sized for a capacity serves every smaller batch), zero-filled before
 * first use (then reused as is).  n < 2^30.  Same errors as the two calls above. */
size_t hs_cascade_step_workspace(int64_t n, int32_t seq_len);
hs_status_t hs_cascade_step(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                            int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                            const int64_t* row_index, const int64_t* d_n, float temperature,
                            hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                            const float* d_threshold, const int64_t* ids, const void* payload, int64_t payload_row_bytes,
                            int64_t* acc_ids, float* acc_conf, int32_t* acc_pred,
                            int64_t* next_ids, void* next_payload, int64_t* d_counts, void* ws,
                            size_t ws_bytes, uint32_t* d_status, hs_stream_t stream);
/* hs_cascade_step_ex: hs_cascade_step plus flags.
 *   HS_STEP_OVERLAP_PREVIOUS: the stage's confidence kernel starts while the
 *   previous libhs kernel on the stream is still running (programmatic
 *   dependent launch without the early wait), e.g. routing stage 0 next to the
 *   latency-bound calibration it does not depend on.  The CALLER guarantees that
 *   the previous libhs call neither writes this step's inputs (logits,
 *   row_index, d_n, ids, payload) nor reads or writes this step's workspace.
 *   Stream order is otherwise preserved: the step's kernels complete after the
 *   previous kernel, and the threshold test waits for it (d_threshold may be
 *   produced by it).
 *   HS_STEP_LOGITS_CAPACITY: `logits` holds all n*seq_len rows (the capacity)
 *   even when d_n makes fewer of them live, so dense rows below the capacity may
 *   be read before the live count is known (the first rows' loads then overlap
 *   the previous libhs kernel's drain).  Without the flag and with d_n, only
 *   live rows are ever read.  Results are identical either way.
 *   Unknown flag bits -> HS_ERR_INVALID_ARGUMENT.
 * top_k: the stage's confidence over its top_k logits (hs_confidence_topk). */
#define HS_STEP_OVERLAP_PREVIOUS 1u
#define HS_STEP_LOGITS_CAPACITY 2u
hs_status_t hs_cascade_step_ex(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                               int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                               const int64_t* row_index, const int64_t* d_n, float temperature,
                               hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                               const float* d_threshold, const int64_t* ids, const void* payload,
                               int64_t payload_row_bytes, int64_t* acc_ids, float* acc_conf,
                               int32_t* acc_pred, int64_t* next_ids, void* next_payload,
                               int64_t* d_counts, void* ws, size_t ws_bytes, uint32_t* d_status,
                               int32_t top_k, uint32_t flags, hs_stream_t stream);

/* The two halves of hs_cascade_step_ex, for callers that take the compaction
 * off the critical path (the next stage's confidence needs only the COUNT of
 * deferred items when its logits are the dense batch of those items):
 *   hs_cascade_confidence: the stage's confidence (K1, + K2 for sequences) into
 *     the step workspace `ws`; with d_defer_count != NULL also ADDS the number
 *     of items the threshold test will defer (0 at the last stage) to
 *     *d_defer_count (caller zero-fills it; same fp32 test as the compaction,
 *     so it equals d_counts[1]).
 *   hs_cascade_compact: the threshold test + stable compaction (+ gather) of
 *     the confidences a previous hs_cascade_confidence left in `ws` (same n,
 *     seq_len, d_n, threshold).  May run on another stream than the next
 *     stage's confidence, ordered after this stage's hs_cascade_confidence; a
 *     workspace is then needed per stage in flight.
 * Arguments as for hs_cascade_step_ex. */
hs_status_t hs_cascade_confidence(int32_t stage, int32_t n_stages, const void* logits, hs_dtype_t dtype,
                                  int64_t n, int32_t seq_len, int64_t n_classes, int64_t row_stride,
                                  const int64_t* row_index, const int64_t* d_n, float temperature,
                                  hs_conf_kind_t kind, hs_seq_reduce_t reduce, float threshold,
                                  const float* d_threshold, uint64_t* d_defer_count, void* ws,
                                  size_t ws_bytes, uint32_t* d_status, int32_t top_k, uint32_t flags,
                                  hs_stream_t stream);
hs_status_t hs_cascade_compact(int32_t stage, int32_t n_stages, int64_t n, int32_t seq_len,
                               const int64_t* d_n, float threshold, const float* d_threshold,
                               const int64_t* ids, const void* payload, int64_t payload_row_bytes,
                               int64_t* acc_ids, float* acc_conf, int32_t* acc_pred, int64_t* next_ids,
                               void* next_payload, int64_t* d_counts, void* ws, size_t ws_bytes,
                               hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Offline Accuracy-Preserving threshold calibration (Alg. 1, AP).  */
/* ------------------------------------------------------------------------ */
/* Deterministic forward-greedy sweep on a 2^q grid (replaces Alg. 1's random
 * sampler, reading G8): bin(c) = min(B, floor(c*B)), B = 2^log2_bins, NaN never
 * accepted.  Round k = 0..K-2 over the validation samples still alive:
 *   G = sum_alive correct[K-1][r];  S(b) = sum_{alive, bin >= b} (correct[k][r] - correct[K-1][r])
 *   b_k = min { b in 0..B+1 : A + G + S(b) >= tau },  A += sum_{alive, bin >= b_k} correct[k][r]
 * t_k = b_k / B, or +inf for b_k = B+1 (defer all); t_{K-1} = 0.  tau = target_correct,
 * or (target_correct < 0, AP) the count of correct answers of m_K.
 * Inputs: conf [(K-1) x N] fp32 (stage k's confidence of sample r at k*N + r),
 * correct [K x N] u8 (0/1).  Outputs (device): d_bin_idx[K-1], d_thresholds[K],
 * d_reach[K], d_handled[K], d_correct_total[1] (int64 counts).
 * log2_bins in [1, 14]; 2 <= K <= 17; N >= 1.  refine_passes (0..64) optional
 * passes after the greedy sweep, each re-picking b_k = min{b : A_k +
 * sum_{alive_k, bin>=b} correct_k + sum_{alive_k, bin<b} C_{k+1} >= tau} for
 * k = 0..K-2 in order, with alive_k / A_k (answers given before k) / C_{k+1}
 * (downstream cascade correctness) under the current thresholds; never raises
 * any b_k; reach / handled / correct_total are then recomputed by a replay.
 * Workspace: hs_calibrate_workspace(K, log2_bins) bytes (no zero-fill needed).
 * Entirely stream-ordered (capturable in a CUDA graph). */
size_t hs_calibrate_workspace(int32_t K, int32_t log2_bins);
hs_status_t hs_calibrate_thresholds(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                    int32_t log2_bins, int64_t target_correct,
                                    int32_t refine_passes, int32_t* d_bin_idx,
                                    float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                    int64_t* d_correct_total, void* ws, size_t ws_bytes,
                                    hs_stream_t stream);

/* Building blocks of the same sweep for request-sharded calibration across
 * GPUs (each rank holds a shard of the validation set; the caller sums the
 * histograms across ranks between the two calls, e.g. with an all-reduce):
 *   hs_calibrate_begin:      zero the histogram/state in ws, set tau (target >= 0) or AP.
 *   hs_calibrate_histogram:  round k: add this shard's 3 x (B+2) int32 histogram
 *                            (count, correct_k, correct_K per bin; index 0 = NaN)
 *                            into hs_calibrate_hist_ptr(ws).
 *   hs_calibrate_select:     round k: pick b_k from the (summed) histogram, update
 *                            A, reach/handled, thresholds; zero the histogram.
 * Every rank that runs select on identical histograms gets identical b_k. */
hs_status_t hs_calibrate_begin(int32_t K, int32_t log2_bins, int64_t target_correct, void* ws,
                               size_t ws_bytes, hs_stream_t stream);
int32_t* hs_calibrate_hist_ptr(void* ws);
size_t hs_calibrate_hist_bytes(int32_t log2_bins);
hs_status_t hs_calibrate_histogram(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                   int32_t log2_bins, int32_t round, const int32_t* d_bin_idx,
                                   void* ws, size_t ws_bytes, hs_stream_t stream);
hs_status_t hs_calibrate_select(int32_t K, int32_t log2_bins, int32_t round, int32_t* d_bin_idx,
                                float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                int64_t* d_correct_total, void* ws, size_t ws_bytes,
                                hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Temperature fitting (NEXT-3; Eq. 1; clamp range S:112).         */
/* ------------------------------------------------------------------------ */
/* For every stage model b (0 <= b < n_batches <= 8), on the SAME labelled
 * validation rows ("learn parameters theta that minimize the NLL between
 * confidence scores and labels Y on the validation dataset"):
 *   T_b = argmin_{t_lo <= T <= t_hi} NLL_b(T),
 *   NLL_b(T) = (1/u_b) sum_{used rows i} [ log sum_j exp(x_ij / T) - x_{i,labels[i]} / T ].
 * logits[b] (host array of device pointers): [n x row_stride] row-major, dtype
 * elements, n_classes valid per row; labels: device int32 [n], shared.  A row
 * is USED iff it is valid (no NaN / +inf, not all -inf) and its label logit is
 * finite with 0 <= label < n_classes; -inf entries are masked classes.  Rows
 * with NaN / +inf (or all -inf) also set HS_STATUS_NONFINITE in *d_status.
 * NLL is convex in beta = 1/T; the minimiser is found by a safeguarded Newton
 * iteration on beta (one pass over the logits per iterate; with n >= 32,768
 * rows of <= 2 KB, up to 2 warm-start Newton sweeps over every 16th row come
 * first; then ~2-4 full passes),
 * converged when a Newton step or the bracket is below 2^-21 relative; a
 * clamp end is returned exactly.  All passes of all stage models run in ONE
 * persistent cooperative kernel launch (one CTA per SM).
 * Outputs (device): d_T[b] fp32 (NaN if no row is used), and optionally
 * d_nll[b] (fp64 mean NLL at the last temperature swept, within the
 * tolerance of d_T[b]), d_passes[b] (full passes at a temperature), d_used[b].
 * max_passes (1..256) bounds the passes; when a model has not converged within
 * it, d_T[b] is the last swept temperature and HS_STATUS_NOT_CONVERGED is ORed
 * into *d_status.  Requires 0 < t_lo <= t_hi < inf.  Workspace:
 * hs_fit_temperature_workspace(n_batches, n) bytes (no zero-fill needed).
 * Errors: INVALID_ARGUMENT (as hs_confidence, plus the range, max_passes and
 * required pointers), WORKSPACE_TOO_SMALL, CUDA (launch failure, e.g. a
 * cooperative launch that cannot be co-resident). */
size_t hs_fit_temperature_workspace(int32_t n_batches, int64_t n);
hs_status_t hs_fit_temperature(const void* const* logits, int32_t n_batches, hs_dtype_t dtype,
                               int64_t n, int64_t n_classes, int64_t row_stride,
                               const int32_t* labels, double t_lo, double t_hi, int32_t max_passes,
                               float* d_T, double* d_nll, int32_t* d_passes, int64_t* d_used,
                               void* ws, size_t ws_bytes, uint32_t* d_status, hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Threshold performance graph, AP and EO (NEXT-4; Alg. 1).        */
/* ------------------------------------------------------------------------ */
/* hs_threshold_replay -- Alg. 1 line 4 ("Compute a on D_v and e = sum_i rho_i
 * e_i") for S threshold vectors at once: the cascade statement
 * replayed on the validation set for each vector.
 *   conf [(K-1) x N] fp32 and correct [K x N] u8 as for hs_calibrate_thresholds;
 *   2 <= K <= 8; log2_bins in [1, 14] (the D5 grid: bin(c) = min(B, floor(c*B)),
 *   NaN never accepted).
 *   d_bvecs: device int32 [S x (K-1)] threshold indices b_k in 0..B+1 (t_k = b_k/B,
 *   B+1 = defer all; values outside are clamped by the compare), or NULL = the
 *   exhaustive grid: S must equal hs_grid_size(K, log2_bins) and vector s has
 *   the digits hs_grid_vector(s) (b_0 most significant).
 *   weights: HOST int64 [K] >= 0, energy of one visit of model k (integer
 *   units, reading G23; rho_k = reach, S:210 / G14).
 * Outputs (device, per vector s): d_correct[s] = correct answers of the
 * cascade, d_energy[s] = sum_k reach_k * weights[k], d_reach[s*K + k]
 * (optional) = requests reaching model k; d_model_correct[k] (optional) = the
 * correct count of model k alone (tau = [K-1] for AP, the EO floor = [K-2]).
 * All exact integers (bit-exact vs the oracle).  S < 2^31, N < 2^32, the
 * energy of a vector < 2^63.  Workspace: hs_threshold_replay_workspace(K, N, log2_bins)
 * (0 for bad K / log2_bins).  The exhaustive grid with B+2 <= 48 (log2_bins <= 5)
 * and N < 2^21 is evaluated through per-prefix histograms of the last
 * threshold's bins ((B+2)x fewer sample visits); results are identical. */
int64_t hs_grid_size(int32_t K, int32_t log2_bins);       /* (B+2)^(K-1), or -1 if >= 2^31 / bad args */
hs_status_t hs_grid_vector(int64_t s, int32_t K, int32_t log2_bins, int32_t* b /* host [K-1] */);
size_t hs_threshold_replay_workspace(int32_t K, int64_t N, int32_t log2_bins);
hs_status_t hs_threshold_replay(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                int32_t log2_bins, const int32_t* d_bvecs, int64_t S,
                                const int64_t* weights, int64_t* d_correct, int64_t* d_energy,
                                int64_t* d_reach, int64_t* d_model_correct, void* ws,
                                size_t ws_bytes, hs_stream_t stream);

/* hs_perf_graph -- the threshold performance graph (the accuracy-vs-energy
 * curve of P:442-444) as its Pareto frontier, and the AP / EO picks.
 *   Input: S points (d_correct[s] in 0..N, d_energy[s] >= 0), e.g. from
 *   hs_threshold_replay.  Frontier: for each correct count c the least energy
 *   of a point with exactly c correct (lowest index on ties), kept iff
 *   strictly below the least energy of every larger count; ascending c (both
 *   c and energy strictly increase).  d_front_c / d_front_e / d_front_s
 *   (capacity N+1) and d_front_n[0] = its length.
 *   AP (G9): d_pick[0] = the least-energy point with >= tau correct
 *   (-1 if none).  EO (G23): d_pick[1] = the interior frontier point
 *   j with c_j >= floor maximising (e_{j+1}-e_j)/(c_{j+1}-c_j) -
 *   (e_j-e_{j-1})/(c_j-c_{j-1}) (fp64, ties to the lowest energy); the AP pick
 *   when no interior point qualifies.
 *   tau / floor_ < 0: taken from d_model_correct[K-1] / [K-2] (required then).
 *   Points with a correct count outside 0..N or a negative energy are ignored
 *   and set HS_STATUS_NONFINITE in *d_status.
 * Workspace: hs_perf_graph_workspace(N). */
size_t hs_perf_graph_workspace(int64_t N);
hs_status_t hs_perf_graph(const int64_t* d_correct, const int64_t* d_energy, int64_t S, int64_t N,
                          int64_t tau, int64_t floor_, const int64_t* d_model_correct, int32_t K,
                          int64_t* d_front_c, int64_t* d_front_e, int64_t* d_front_s,
                          int64_t* d_front_n, int64_t* d_pick, void* ws, size_t ws_bytes,
                          uint32_t* d_status, hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Multi-GPU cascade over peer memory (§V-A; P:561 DMA, P:617-619   */
/* zero-copy): a group of ranks (one process per GPU) that exchange through   */
/* each other's memory over NVLink / NVSwitch, with no host round trip and no */
/* NCCL on the data path.                                                    */
/* ------------------------------------------------------------------------ */
/* Every rank g owns one PEER REGION of hs_peer_region_bytes(world, cap, P, q)
 * bytes, allocated with hs_ipc_alloc (zero-filled, exportable); the 64-byte
 * hs_ipc_handle of every region is exchanged once by the caller (e.g.
 * torch.distributed all_gather_object) and opened with hs_ipc_open, so that
 * hs_peer_t.region[h] is rank h's region as mapped in this process
 * (region[rank] = this rank's own allocation).  The region holds the forward
 * flags, two receive sets of world*cap ids (+ payload rows of P bytes) and two
 * calibration slot sets of world x (2^q + 2) packed bins.
 *   cap: the largest batch any rank routes in any stage (every rank's deferred
 *        count must stay <= cap; more sets HS_STATUS_OVERFLOW and is clamped).
 *   All ranks must call the same sequence of hs_peer_* / *_peer operations
 *   (the flags carry per-rank epochs kept on the device).
 *
 * hs_peer_forward -- after a stage every rank g holds D_g deferred ids in
 * increasing global order (next_ids of hs_cascade_step, count *d_count).  The
 * next stage's batch is the global rank-major list, split into contiguous
 * blocks over the destination ranks dest_ranks[0..n_dest) (distinct; NULL =
 * all ranks in order, the balanced placement): block d = global positions
 * [floor(d*D/n_dest), floor((d+1)*D/n_dest)), D = sum_g D_g.  Receiver
 * dest_ranks[d] gets its block, in global order, at hs_peer_recv_ids(g, set)
 * [0 .. *d_recv_count) (and its payload rows at hs_peer_recv_payload(g, set);
 * payload may be NULL).  Three stream-ordered kernels, graph-capturable:
 *   publish: {epoch, D_g} into slot g of every rank's count array;
 *   scatter: wait for every rank's count of the epoch, write each local id
 *            (one thread per item: coalesced peer stores) and payload row at
 *            its final position in the destination's receive set, then (last
 *            CTA) this rank's receive count and a "done" flag to every rank;
 *   wait:    until every rank's done flag carries the epoch.
 *   set (0/1): the receive set written; alternate it between consecutive
 *   forwards (stage parity) -- a rank may scatter stage k+1 while a peer still
 *   reads stage k's set.  The phases are also exported separately (publish all
 *   ranks, then scatter, then wait) for several ranks driven by one process.
 * Waits give up after 10 s (a peer that never publishes): HS_STATUS_TIMEOUT is
 * ORed into *d_status (optional), the receive count is 0, nothing hangs.
 *
 * hs_calibrate_thresholds_peer -- hs_calibrate_thresholds where conf / correct
 * hold THIS rank's shard (N >= 0 samples, may be 0): every round, each rank's
 * packed histogram is pushed into every rank's region inside the one
 * cooperative calibration kernel (system-scope release counter), and every
 * rank selects the identical b_k from the sum of the W histograms (integer
 * counts: order-independent, deterministic).  AP: tau = the GLOBAL correct
 * count of m_K.  Needs q = the group's log2_bins, K <= 16, N * world < 2^21
 * and a shard that fits the resident kernel (else HS_ERR_UNSUPPORTED, before
 * any launch).  No refinement passes on this path.
 *
 * hs_cascade_step_peer -- hs_cascade_step_ex, then (stage < n_stages-1)
 * hs_peer_forward of its next_ids / next_payload / d_counts[1] to
 * next_stage_ranks (SURVEY 8(b)'s comm-aware cascade step).  n must be <= cap.
 *
 * hs_ipc_alloc / hs_ipc_free: the one explicit device allocation of the library
 * (a whole cudaMalloc allocation, zero-filled synchronously, so that its IPC
 * handle maps exactly this buffer on the peers).
 * hs_ipc_handle / hs_ipc_open / hs_ipc_close wrap cudaIpcGetMemHandle /
 * cudaIpcOpenMemHandle (lazy peer access) / cudaIpcCloseMemHandle. */
#define HS_PEER_MAX_WORLD 8
typedef struct {
  int32_t rank, world;                /* 0 <= rank < world <= 8 */
  int64_t cap;                        /* max items per rank per stage (< 2^32) */
  int64_t payload_row_bytes;          /* 0 or a multiple of 16 */
  int32_t log2_bins;                  /* calibration grid the regions are sized for (1..14) */
  void* region[HS_PEER_MAX_WORLD];    /* region[h]: rank h's region, mapped in this process */
} hs_peer_t;
size_t hs_peer_region_bytes(int32_t world, int64_t cap, int64_t payload_row_bytes, int32_t log2_bins);
int64_t* hs_peer_recv_ids(const hs_peer_t* g, int32_t set);     /* this rank's receive set (device) */
void* hs_peer_recv_payload(const hs_peer_t* g, int32_t set);    /* NULL without payload rows */
hs_status_t hs_peer_forward(const hs_peer_t* g, int32_t set, const int64_t* ids, const void* payload,
                            const int64_t* d_count, const int32_t* dest_ranks, int32_t n_dest,
                            int64_t* d_recv_count, uint32_t* d_status, hs_stream_t stream);
hs_status_t hs_peer_forward_publish(const hs_peer_t* g, const int64_t* d_count, uint32_t* d_status,
                                    hs_stream_t stream);
hs_status_t hs_peer_forward_scatter(const hs_peer_t* g, int32_t set, const int64_t* ids, const void* payload,
                                    const int32_t* dest_ranks, int32_t n_dest, int64_t* d_recv_count,
                                    uint32_t* d_status, hs_stream_t stream);
hs_status_t hs_peer_forward_wait(const hs_peer_t* g, uint32_t* d_status, hs_stream_t stream);
hs_status_t hs_calibrate_thresholds_peer(const float* conf, const uint8_t* correct, int32_t K, int64_t N,
                                         int32_t log2_bins, int64_t target_correct, int32_t* d_bin_idx,
                                         float* d_thresholds, int64_t* d_reach, int64_t* d_handled,
                                         int64_t* d_correct_total, const hs_peer_t* g, void* ws,
                                         size_t ws_bytes, uint32_t* d_status, hs_stream_t stream);
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
                                 int64_t* d_recv_count, hs_stream_t stream);
hs_status_t hs_ipc_alloc(size_t bytes, void** dptr);   /* cudaMalloc + zero fill: exportable whole allocation */
hs_status_t hs_ipc_free(void* dptr);
hs_status_t hs_ipc_handle(const void* dptr, void* handle /* host, 64 bytes */);
hs_status_t hs_ipc_open(const void* handle /* host, 64 bytes */, void** dptr);
hs_status_t hs_ipc_close(void* dptr);

/* ------------------------------------------------------------------------ */
/* Request-sharded calibration across GPUs with the library's own NCCL        */
/* communicator.                                          */
/* ------------------------------------------------------------------------ */
/* hs_comm_unique_id: rank 0 creates a 128-byte NCCL unique id (host) and
 *   shares it with the other ranks (e.g. over torch.distributed).
 * hs_comm_create: every rank joins with the shared id (collective over the
 *   group; blocks until all ranks joined).  The library owns the handle.
 * hs_calibrate_thresholds_comm: hs_calibrate_thresholds where conf / correct
 *   hold THIS rank's shard of the validation set (N = local samples): per round
 *   every rank histograms its shard, the int32 histograms are summed with an
 *   NCCL all-reduce on `stream`, and every rank selects the identical b_k from
 *   the global histogram (integer counts: order-independent, deterministic).
 *   target_correct < 0: AP, tau = the GLOBAL correct count of m_K.  comm ==
 *   NULL: single GPU (the same sweep without the all-reduce).  Outputs as
 *   hs_calibrate_thresholds (refinement passes: hs_calibrate_thresholds_comm_ex).
 *   Every argument is validated before the first collective, so an argument
 *   error returns on the failing rank before any rank has entered a round
 *   (the arguments that decide the collectives -- K, log2_bins -- must agree
 *   across ranks).  NCCL failures: HS_ERR_NCCL.
 * NCCL is loaded with dlopen("libnccl.so.2") on the first of these calls;
 * HS_ERR_UNSUPPORTED when it cannot be loaded. */
typedef struct hs_comm_s* hs_comm_t;
/* hs_forward_nccl -- the NCCL path of the forwarding step (
 * hs_forward_* is the peer-memory path): after hs_cascade_step on every rank,
 * move this rank's deferred ids[0..*d_count) (+ payload rows of
 * payload_row_bytes) so that dest_ranks[d] (distinct) receives block d of the
 * global rank-major deferred list (as hs_forward_scatter / dist.forward_deferred).
 * One all-gather of every rank's (count, recv_cap), ONE device->host read of
 * them (NCCL sizes are host values: this call synchronises `stream`), then
 * grouped ncclSend/ncclRecv.  recv_ids / recv_payload hold recv_cap rows;
 * *h_recv_count (host) = rows received.  When ANY rank's block exceeds that
 * rank's recv_cap, EVERY rank returns HS_ERR_INVALID_ARGUMENT after the
 * all-gather and none posts a send or receive (the decision is taken on the
 * gathered values, so no rank is left waiting).  NCCL failures: HS_ERR_NCCL.
 * ws: hs_forward_nccl_workspace(world) bytes of device memory. */
size_t hs_forward_nccl_workspace(int32_t world);
hs_status_t hs_forward_nccl(const int64_t* ids, const void* payload, int64_t payload_row_bytes,
                            const int64_t* d_count, const int32_t* dest_ranks, int32_t n_dest,
                            int64_t* recv_ids, void* recv_payload, int64_t recv_cap,
                            int64_t* h_recv_count, hs_comm_t comm, void* ws, size_t ws_bytes,
                            hs_stream_t stream);
hs_status_t hs_comm_unique_id(void* id /* host, 128 bytes */);
hs_status_t hs_comm_create(const void* id /* host, 128 bytes */, int32_t rank, int32_t world,
                           int32_t device, hs_comm_t* out);
hs_status_t hs_comm_destroy(hs_comm_t comm);
hs_status_t hs_calibrate_thresholds_comm(const float* conf, const uint8_t* correct, int32_t K,
                                         int64_t N, int32_t log2_bins, int64_t target_correct,
                                         int32_t* d_bin_idx, float* d_thresholds, int64_t* d_reach,
                                         int64_t* d_handled, int64_t* d_correct_total,
                                         hs_comm_t comm, void* ws, size_t ws_bytes,
                                         hs_stream_t stream);
/* hs_calibrate_thresholds_comm_ex: the same plus refine_passes (0..64) D5
 * refinement passes on the sharded set (as hs_calibrate_thresholds): per pass
 * and stage the refinement histogram and A_k are summed across ranks, and the
 * final replay's reach / handled / correct_total are summed too. */
hs_status_t hs_calibrate_thresholds_comm_ex(const float* conf, const uint8_t* correct, int32_t K,
                                            int64_t N, int32_t log2_bins, int64_t target_correct,
                                            int32_t refine_passes, int32_t* d_bin_idx, float* d_thresholds,
                                            int64_t* d_reach, int64_t* d_handled, int64_t* d_correct_total,
                                            hs_comm_t comm, void* ws, size_t ws_bytes, hs_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Diagnostics.                                                              */
/* ------------------------------------------------------------------------ */
const char* hs_status_string(hs_status_t s);
const char* hs_last_error(void);     /* thread-local detail of the last failure */
uint64_t hs_launch_count(void);      /* kernels this process has launched through libhs */
const char* hs_build_info(void);     /* compile target / flags */

#ifdef __cplusplus
}
#endif
#endif /* HS_H_ */
