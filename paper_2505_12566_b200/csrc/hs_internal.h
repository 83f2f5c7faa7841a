// hs_internal.h -- launcher interfaces between the C-ABI layer (api.cu) and the
// kernels (conf.cu, compact.cu, calib.cu).  Not part of the public ABI.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <utility>

#include "../../include/hs.h"

struct hs_comm_s;

namespace hs {

int num_sms();          // SM count of the current device (cached per device)
void count_launch();    // bumps the process-wide launch counter (hs_launch_count)
bool pdl_enabled();     // programmatic dependent launch (HS_NO_PDL=1 disables)

// Every libhs kernel is launched with programmatic dependent launch: the next
// kernel of the stream is scheduled while this one drains, and waits with
// griddepcontrol.wait (pdl_wait) before touching the previous kernel's output.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t s, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = pdl_enabled() ? 1 : 0;
  const cudaError_t e = cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
  count_launch();
  return e != cudaSuccess ? e : cudaGetLastError();
}

// ---- K1 / K2 ---------------------------------------------------------------
constexpr int kMaxBatch = 8;
// K1 with the stage's threshold test and stable compaction (K3) fused into it
// (hs_cascade_step with HS_FUSE=1, single-token rows on the cp.async kernel):
// per-tile deferred counters while the rows stream, one grid barrier, then the
// prefixes and the lists (conf.cu).
constexpr int kFuseTiles = 1024;
struct FuseArgs {
  int on;                         // 0: plain K1
  int is_last;                    // the last stage accepts every row
  float threshold;
  const float* d_threshold;       // overrides threshold when non-NULL
  const int64_t* ids;             // request id of row i, or NULL (= i)
  int64_t* acc_ids;               // accepted: id, confidence, argmax (stable order)
  float* acc_conf;
  int32_t* acc_pred;
  int64_t* def_ids;               // deferred: id (the next stage's batch), stable order
  int64_t* def_pos;               // deferred: row position (payload gather), or NULL
  int64_t* counts;                // {n_acc, n_def}
  void* tiles;                    // fuse_ws_bytes(): epoch, two banks of tile counters
};
constexpr size_t fuse_ws_bytes() { return 32 + (size_t)kFuseTiles * 8; }
struct ConfArgs {
  const void* logits;
  int64_t row_bytes;       // row_stride * element size (multiple of 16)
  int64_t n;               // batch items (capacity when d_n != NULL)
  int L;                   // tokens per item
  int64_t C;               // classes
  int nvec;                // 16-byte vectors covering C elements
  int tail;                // C % elements-per-vector (0: last vector full)
  const int64_t* row_index;
  const int64_t* d_n;
  float c;                 // log2(e) / T
  int kind;                // hs_conf_kind_t
  float* conf;             // [n*L] per token row
  int32_t* argmax;         // [n*L] or NULL
  const int32_t* labels;   // indexed by source token row, or NULL
  uint8_t* ok;             // [n*L] argmax == label, or NULL
  uint32_t* status;        // or NULL
  // batched stages (hs_confidence_batched): output rows [b*brows, (b+1)*brows)
  // read batch b's logits bptr[b] at temperature factor bc[b]
  int nbatch;              // 1 = plain call (logits, c)
  int64_t brows;           // n * L rows per batch
  uint64_t bmagic;         // ceil(2^64 / brows): row / brows = umul64hi(row, bmagic) for
                           // row < 2^32 (brows >= 2; brows == 1 -> 0, quotient = row)
  const void* bptr[kMaxBatch];
  float bc[kMaxBatch];
  // async kernel only: rows claimed in warp-sized groups from ticket[0] (reset
  // to 0 by the last CTA through ticket[1]); NULL = static grid-stride rows
  unsigned int* ticket;
  // async kernel only: read the inputs without waiting for the previous kernel
  // of the stream, wait for it just before exiting (stream order preserved)
  int late_wait;
  // NEXT-2: softmax restricted to the top_k largest logits (0 = full row)
  int top_k;
  // K1e split rows (small batches of long rows): zero-filled-once workspace of
  // split_ws_bytes(rows) bytes, or NULL (no split)
  void* split_ws;
  int split_zero;          // 1: zero the arrival counters before the launch
  // optional second output: exp(-H) of every row alongside `conf` (north_star
  // "max-probability (and entropy) confidence"); forces the entropy sums
  float* conf2;
  // K1+K3 fused (async kernel with a ticket, L = 1, nbatch = 1, no late wait)
  FuseArgs fz;
  // the LAST stage of a cascade (it accepts every row, so its compaction is the
  // identity): K1 writes conf / argmax straight into the accepted lists, copies
  // the ids (NULL: the row) into last_ids_out and writes {live rows, 0} into
  // last_counts -- no K3 launch (hs_cascade_step, L = 1)
  const int64_t* last_ids;
  int64_t* last_ids_out;
  int64_t* last_counts;
  // the logits hold all n * L * nbatch rows (true without d_n; with d_n the
  // caller says so, HS_STEP_LOGITS_CAPACITY): dense rows may be read before the
  // previous kernel's live count is visible
  int rows_cap_valid;
};
// true when launch_confidence(a) takes the cp.async kernel, which is the one
// that can run the fused threshold test + compaction
bool confidence_fusable(const ConfArgs& a);
constexpr int kSplitMaxRows = 2048;     // the split path serves batches up to this many rows
constexpr int kSplitMaxSeg = 64;        // segments per row
size_t split_ws_bytes(int64_t rows);
constexpr int kTopkMax = 32;
cudaError_t launch_confidence(const ConfArgs& a, bool bf16, cudaStream_t s);
cudaError_t launch_seq_reduce(const float* tok_conf, const uint8_t* tok_ok, int64_t n,
                              const int64_t* d_n, int L, int reduce, float* conf,
                              uint8_t* correct, cudaStream_t s);
const char* confidence_path(int64_t nvec);

// ---- K3 / K4 ---------------------------------------------------------------
constexpr int kCompactThreads = 256;
constexpr int kCompactItems = 8;
constexpr int kCompactTile = kCompactThreads * kCompactItems;   // 2048 items per tile

struct CompactWs {          // zero-filled before first use; then self-maintaining
  unsigned int epoch;       // launch counter tagging the tile descriptors
  unsigned int ticket;      // tile tickets: CTAs take tiles in the order they START
  unsigned long long pad[3];
  // unsigned long long status[n_tiles] follows (32-byte header)
};
size_t compact_ws_bytes(int64_t n);
cudaError_t launch_count_deferred(const float* conf, int64_t cap, const int64_t* d_n, float threshold,
                                  const float* d_threshold, int is_last, unsigned long long* out,
                                  cudaStream_t s);

struct CompactArgs {
  const float* conf;
  int64_t n;
  const int64_t* d_n;
  float threshold;
  const float* d_threshold;   // overrides threshold when non-NULL
  int is_last;
  const int64_t* ids;
  const int32_t* pred;
  int pred_len;
  int64_t* acc_ids;
  float* acc_conf;
  int32_t* acc_pred;
  int64_t* def_ids;
  int64_t* def_pos;
  int64_t* counts;
  void* ws;
  // selection mode (skip connections): select items i with sel_dest[i] == sel_k
  const int32_t* sel_dest;
  int sel_k;
  // skip-route mode: write skip_dest[ids[i]] = next model (or K + stage when answered)
  int32_t* skip_dest;
  int skip_K;
  int skip_stage;
  int skip_mode;         // 0 uniform, 1 decade ("LogUniform")
};
constexpr int kMaxSkipEdges = 15;
cudaError_t launch_route_compact(const CompactArgs& a, cudaStream_t s);
cudaError_t launch_gather_rows(const int64_t* pos, const int64_t* d_count, int64_t cap,
                               const void* src, int64_t row_bytes, void* dst, cudaStream_t s);

// ---- K5 / K6 ---------------------------------------------------------------
struct CalibState {         // lives at the start of the calibration workspace
  long long A;              // correct answers committed so far
  long long tau;            // target correct count
  int tau_ap;               // 1: tau = correct count of m_K (set in round 0)
  int pad[11];
};
size_t calib_hist_bytes(int q);
size_t calib_ws_bytes(int K, int q);
cudaError_t launch_calib_init(void* ws, int q, long long target, cudaStream_t s);
cudaError_t launch_calib_refine_round(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                                      int k, const int32_t* b_idx, void* ws, bool zero_hist, cudaStream_t s);
cudaError_t launch_calib_replay(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                                const int32_t* b_idx, int64_t* reach, int64_t* handled, int64_t* correct_total,
                                cudaStream_t s);
cudaError_t launch_calib_hist(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                              int round, const int32_t* b_idx, int32_t* hist, cudaStream_t s);
cudaError_t launch_calib_fused(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                               long long target, int32_t* b_idx, float* thr, int64_t* reach,
                               int64_t* handled, int64_t* correct_total, void* ws, cudaStream_t s);
cudaError_t launch_calib_cluster(const float* conf, const uint8_t* correct, int K, int64_t N,
                                 int q, long long target, int32_t* b_idx, float* thr,
                                 int64_t* reach, int64_t* handled, int64_t* correct_total,
                                 void* ws, cudaStream_t s);
cudaError_t launch_calib_refine(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                                int passes, int32_t* b_idx, float* thr, int64_t* reach,
                                int64_t* handled, int64_t* correct_total, void* ws, cudaStream_t s);
cudaError_t launch_calib_select(int K, int q, int round, int32_t* b_idx, float* thr,
                                int64_t* reach, int64_t* handled, int64_t* correct_total,
                                void* ws, cudaStream_t s);

// ---- NEXT-3: temperature fitting (Eq. 1) ------------------------------------
constexpr int kTfMaxGrid = 1024;   // CTAs of the persistent launch (partials sized for it)
struct TfArgs {
  const void* bptr[kMaxBatch];     // stage b's validation logits
  int nbatch;                      // stage models fitted together
  int64_t n;                       // rows per stage
  int64_t row_bytes;               // row_stride * element size (multiple of 16)
  int64_t C;                       // classes
  int nvec, tail;                  // 16-byte vectors per row, C % elements-per-vector
  const int32_t* labels;           // [n], shared by every stage
  double blo0, bhi0;               // beta = 1/T range [1/t_hi, 1/t_lo]
  double t_lo, t_hi;               // clamp range of T (returned exactly at a clamp)
  double tol;                      // relative Newton-step / bracket tolerance on beta
  int max_passes;                  // sweeps at a temperature (after the max sweep)
  float2* rowstat;                 // ws: [nbatch * n] {m, x_y - m}; m = NaN: row unused
  double* partial;                 // ws: [2][grid][nbatch][3]
  float* T;                        // [nbatch] fitted temperatures
  double* nll;                     // [nbatch] mean NLL at the last swept temperature, or NULL
  int32_t* passes;                 // [nbatch] sweeps used, or NULL
  int64_t* used;                   // [nbatch] rows in the mean, or NULL
  uint32_t* status;                // or NULL
};
size_t temp_fit_ws_bytes(int nbatch, int64_t n);
cudaError_t launch_temp_fit(TfArgs a, bool bf16, void* ws, cudaStream_t s);

// ---- NEXT-4: threshold performance graph (Alg. 1) ---------------------------
constexpr int kReplayMaxK = 8;
struct ReplayWeights {
  unsigned long long cum[kReplayMaxK];   // cum[j] = sum_{k <= j} w_k: energy of a request answered by m_j
};
struct ReplayArgs {
  int K;                    // models (2..kReplayMaxK)
  int64_t N;                // validation samples
  int64_t Np;               // N rounded up to 4 (set by launch_replay)
  int q;                    // log2 bins
  const int32_t* bvecs;     // [S x (K-1)] grid indices, or NULL = the exhaustive grid
  int64_t S;                // threshold vectors
  ReplayWeights w;
  int32_t* bins;            // ws: [(K-1) x Np]
  uint32_t* bits;           // ws: [Np] correct bits
  int64_t* out_c;           // [S] correct counts
  int64_t* out_e;           // [S] energies
  int64_t* reach;           // [S x K] or NULL
};
size_t replay_ws_bytes(int K, int64_t N, int q);
cudaError_t launch_replay(ReplayArgs a, const float* conf, const uint8_t* correct,
                          unsigned long long* model_correct, void* ws, cudaStream_t s);
size_t graph_ws_bytes(int64_t N);
cudaError_t launch_graph(const int64_t* C, const int64_t* E, int64_t S, int64_t N, int64_t tau,
                         int64_t floor_, const unsigned long long* model_correct, int K,
                         int64_t* front_c, int64_t* front_e, int64_t* front_s, int64_t* front_n,
                         int64_t* pick, uint32_t* status, void* ws, cudaStream_t s);

// ---- multi-GPU exchange over peer memory (peer.cu; calib.cu's resident kernel) --
constexpr int kPeerMaxWorld = 8;
struct PeerHeader {                 // start of every rank's peer region
  unsigned long long fwd_counts[kPeerMaxWorld];   // slot g: {epoch:32 | count:32} from rank g
  unsigned long long fwd_done[kPeerMaxWorld];     // slot g: epoch from rank g
  unsigned long long cal_arrive[2];               // calibration pushes received, per round parity
  unsigned fwd_epoch, fwd_ctr, fwd_failed, pad0;  // local: forward epoch, completion counter, timeout flag
  unsigned long long cal_round;                   // local: calibration rounds run so far
  unsigned long long pad[10];
};
struct PeerLayout {                 // byte offsets inside a region (identical on every rank)
  size_t cal_off, cal_words, recv_off, recv_stride, pay_off, bytes;
};
PeerLayout peer_layout(int world, int64_t cap, int64_t payload_row_bytes, int q);
struct PeerArgs {                   // the group as seen by this process
  int world, rank;
  int64_t recv_stride;                            // rows per receive set (world * cap)
  PeerHeader* hdr[kPeerMaxWorld];                 // rank h's region header
  int64_t* recv_ids[kPeerMaxWorld];               // rank h's receive sets [2][recv_stride]
  void* recv_payload[kPeerMaxWorld];              // rank h's payload sets [2][recv_stride][P] (or NULL)
};
struct PeerDest {
  int n;                                          // destination ranks of the next stage
  int ranks[kPeerMaxWorld];
};
struct PeerCal {                    // calibration exchange of calib_resident_kernel
  int world, rank;
  unsigned long long* slots[kPeerMaxWorld];       // rank h's cal slots [2][world][2^q + 2]
  unsigned long long* arrive[kPeerMaxWorld];      // rank h's cal_arrive[2]
  unsigned long long* round_ctr;                  // this rank's cal_round
  uint32_t* status;
};
cudaError_t launch_peer_publish(const int64_t* d_count, int64_t cap, const PeerArgs& g, uint32_t* status,
                                cudaStream_t s);
cudaError_t launch_peer_scatter(const int64_t* ids, const void* payload, int64_t row_bytes, int64_t cap,
                                int set, const PeerArgs& g, const PeerDest& dest, int64_t* d_recv_count,
                                uint32_t* status, cudaStream_t s);
cudaError_t launch_peer_wait(const PeerArgs& g, uint32_t* status, cudaStream_t s);
cudaError_t launch_calib_peer(const float* conf, const uint8_t* correct, int K, int64_t N, int q,
                              long long target, int32_t* b_idx, float* thr, int64_t* reach,
                              int64_t* handled, int64_t* correct_total, void* ws, const PeerCal& pc,
                              cudaStream_t s);

// ---- NCCL communicator (comm.cu; NCCL is dlopen-ed on first use) ---------------
bool nccl_available();
const char* nccl_error(int r);
int nccl_unique_id(void* out128);
int nccl_comm_create(const void* id128, int rank, int world, int device, hs_comm_s** out);
int nccl_comm_destroy(hs_comm_s* c);
int nccl_allreduce_i32_sum(int32_t* buf, size_t count, hs_comm_s* c, cudaStream_t s);
int nccl_allreduce_i64_sum(int64_t* buf, size_t count, hs_comm_s* c, cudaStream_t s);
int nccl_world(const hs_comm_s* c);
int nccl_rank(const hs_comm_s* c);
int nccl_allgather_i64(const int64_t* mine, int64_t* all, int64_t count, hs_comm_s* c, cudaStream_t s);
int nccl_exchange(const char* sbuf, const int64_t* soff, const int64_t* scnt, char* rbuf,
                  const int64_t* roff, const int64_t* rcnt, int64_t elem_bytes, hs_comm_s* c,
                  cudaStream_t s);

}  // namespace hs
