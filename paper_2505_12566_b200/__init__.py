"""HybridServe cascade router on B200 (sm_100a) -- thin Python binding of libhs.so.

Every step of the router (confidence, threshold test, compaction, gather,
calibration) runs in the CUDA kernels behind the C-ABI of ``include/hs.h``;
this module only turns torch tensors into pointers, allocates caller-owned
buffers with torch, and passes ``torch.cuda.current_stream()``.  There is no
CPU fallback: without ``libhs.so`` (or a GPU) every call raises.

Names follow the C-ABI (``hs_confidence`` -> ``confidence`` ...).  The paper's
statement of the cascade: models m_1..m_K, small to large, with
thresholds t_1..t_{K-1}; a request answered by m_k iff its confidence at m_k
is >= t_k; t_K = 0.
"""
from __future__ import annotations

import dataclasses

import torch

from . import _abi
from ._abi import HsError, lib

MAXPROB, MAXPROB_SQ, ENTROPY = 0, 1, 2
SEQ_NONE, SEQ_MIN, SEQ_MEAN = 0, 1, 2
HS_STEP_OVERLAP_PREVIOUS = 1     # hs_cascade_step_ex flags (include/hs.h)
HS_STEP_LOGITS_CAPACITY = 2


def _rows_capacity_flag(logits: torch.Tensor, rows: int, row_index) -> int:
    """HS_STEP_LOGITS_CAPACITY when the memory from ``logits``' first row on
    holds ``rows`` rows of its stride (e.g. a view of the live rows of a
    capacity-sized buffer), so dense rows below the capacity may be read before
    the live count is known."""
    if row_index is not None or logits.dim() != 2:
        return 0
    eb = logits.element_size()
    avail = logits.untyped_storage().nbytes() - logits.storage_offset() * eb
    need = (rows - 1) * logits.stride(0) * eb + logits.shape[1] * eb if rows > 0 else 0
    return HS_STEP_LOGITS_CAPACITY if avail >= need else 0
_KINDS = {"maxprob": MAXPROB, "maxprob_sq": MAXPROB_SQ, "entropy": ENTROPY}
_REDUCES = {"none": SEQ_NONE, "min": SEQ_MIN, "mean": SEQ_MEAN}
STATUS_NONFINITE = 1
STATUS_NOT_CONVERGED = 2
STATUS_TIMEOUT = 4

__all__ = ["confidence", "confidence_batched", "route_compact", "cascade_step", "calibrate_thresholds",
           "calibrate_begin", "calibrate_histogram", "calibrate_select", "fit_temperature", "threshold_replay", "perf_graph", "grid_size", "grid_vector",
           "Cascade", "HsError",
           "launch_count", "MAXPROB", "MAXPROB_SQ", "ENTROPY", "SEQ_NONE", "SEQ_MIN", "SEQ_MEAN"]


def _kind(k):
    return _KINDS[k] if isinstance(k, str) else int(k)


def _reduce(r):
    return _REDUCES[r] if isinstance(r, str) else int(r)


def _p(t):
    return None if t is None else t.data_ptr()


def _stream(stream=None):
    s = stream if stream is not None else torch.cuda.current_stream()
    return s.cuda_stream


def _dtype_code(t: torch.Tensor) -> int:
    if t.dtype == torch.bfloat16:
        return 1
    if t.dtype == torch.float32:
        return 0
    raise TypeError(f"logits must be bfloat16 or float32, got {t.dtype}")


def _check_cuda(*ts):
    for t in ts:
        if t is not None and not t.is_cuda:
            raise ValueError("libhs takes CUDA tensors only (no CPU fallback)")


def launch_count() -> int:
    """Kernels launched through libhs by this process."""
    return int(lib().hs_launch_count())


def build_info() -> str:
    return lib().hs_build_info().decode()


def _temp_workspace(nbytes: int, device, stream=None) -> torch.Tensor:
    """A call-local workspace; when the call runs on another stream than torch's
    current one, the caching allocator is told so (record_stream) and does not
    hand the memory out again before that stream is done with it."""
    t = torch.empty(max(int(nbytes), 16), dtype=torch.uint8, device=device)
    if stream is not None and stream != torch.cuda.current_stream(device):
        t.record_stream(stream)
    return t


def workspace(nbytes: int, device) -> torch.Tensor:
    """A zero-filled workspace (the compaction descriptors must start zeroed)."""
    return torch.zeros(max(int(nbytes), 16), dtype=torch.uint8, device=device)


# ---------------------------------------------------------------------------
# hs_confidence
# ---------------------------------------------------------------------------
def confidence(logits: torch.Tensor, *, n: int | None = None, seq_len: int = 1,
               n_classes: int | None = None, temperature: float = 1.0, kind="maxprob",
               reduce="none", row_index: torch.Tensor | None = None,
               d_n: torch.Tensor | None = None, labels: torch.Tensor | None = None,
               want_argmax: bool = True, status: torch.Tensor | None = None,
               out: dict | None = None, ws: torch.Tensor | None = None, top_k: int = 0,
               want_entropy: bool = False, stream=None) -> dict:
    """Per-item confidence of a batch of logits rows.

    ``logits``: [rows, row_stride] bf16/fp32 on the GPU (row-major; the first
    ``n_classes`` entries of a row are the prediction vector).  Returns dict of
    ``conf`` f32[n], ``argmax`` i32[n*seq_len] and ``correct`` u8[n] (when
    ``labels`` is given).  ``top_k`` > 0: softmax restricted to each row's
    top_k logits (NEXT-2; hs_confidence_topk).  ``want_entropy``:
    also ``conf_entropy`` f32[n] = exp(-H) of every row, in the same pass
    (hs_confidence_ex; seq_len 1)."""
    _check_cuda(logits, row_index, d_n, labels, status)
    if logits.dim() != 2 or logits.stride(1) != 1:
        raise ValueError("logits must be a 2-D row-major tensor")
    C = int(n_classes or logits.shape[1])
    stride = int(logits.stride(0))
    if n is None:
        n = int(row_index.numel()) if row_index is not None else logits.shape[0] // seq_len
    dev = logits.device
    out = dict(out or {})
    if "conf" not in out:
        out["conf"] = torch.empty(n, dtype=torch.float32, device=dev)
    if want_argmax and "argmax" not in out:
        out["argmax"] = torch.empty(n * seq_len, dtype=torch.int32, device=dev)
    if labels is not None and "correct" not in out:
        out["correct"] = torch.empty(n, dtype=torch.uint8, device=dev)
    if want_entropy and "conf_entropy" not in out:
        out["conf_entropy"] = torch.empty(n, dtype=torch.float32, device=dev)
    # required: the token-row part (hs_confidence_batched_workspace(1, ..)); a
    # caller workspace of at least that size is used as is (the optional
    # split-row region only when it fits).  A temporary gets the full size.
    need = lib().hs_confidence_batched_workspace(1, n, seq_len)
    if ws is None or ws.numel() < need:
        full = lib().hs_confidence_workspace(n, seq_len)
        ws = _temp_workspace(full, dev, stream) if full else None
    _abi.call("hs_confidence_ex", _p(logits), _dtype_code(logits), n, seq_len, C, stride,
              _p(row_index), _p(d_n), float(temperature), _kind(kind), _reduce(reduce), int(top_k),
              _p(out["conf"]), _p(out.get("conf_entropy")), _p(out.get("argmax")), _p(labels),
              _p(out.get("correct")), _p(ws), 0 if ws is None else ws.numel(), _p(status),
              _stream(stream))
    return out


def confidence_batched(logits: list, temperatures, *, n: int | None = None, seq_len: int = 1,
                       n_classes: int | None = None, kind="maxprob", reduce="none",
                       row_index: torch.Tensor | None = None,
                       labels: torch.Tensor | None = None, want_argmax: bool = True,
                       status: torch.Tensor | None = None, out: dict | None = None,
                       ws: torch.Tensor | None = None, stream=None) -> dict:
    """Every stage model's confidence on the same items in ONE launch (the
    calibration input of Alg. 1).  Output rows b*n .. b*n+n-1 of
    ``conf`` / ``correct`` belong to logits[b]."""
    import ctypes
    nb = len(logits)
    x0 = logits[0]
    _check_cuda(*logits, row_index, labels, status)
    for x in logits:
        if x.dim() != 2 or x.stride(1) != 1 or x.stride(0) != x0.stride(0) or x.dtype != x0.dtype:
            raise ValueError("batched logits must share dtype, shape and row stride")
    C = int(n_classes or x0.shape[1])
    if n is None:
        n = int(row_index.numel()) if row_index is not None else x0.shape[0] // seq_len
    dev = x0.device
    out = dict(out or {})
    if "conf" not in out:
        out["conf"] = torch.empty(nb * n, dtype=torch.float32, device=dev)
    if want_argmax and "argmax" not in out:
        out["argmax"] = torch.empty(nb * n * seq_len, dtype=torch.int32, device=dev)
    if labels is not None and "correct" not in out:
        out["correct"] = torch.empty(nb * n, dtype=torch.uint8, device=dev)
    need = lib().hs_confidence_batched_workspace(nb, n, seq_len)
    if need and (ws is None or ws.numel() < need):
        ws = _temp_workspace(need, dev, stream)
    ptrs = (ctypes.c_void_p * nb)(*[x.data_ptr() for x in logits])
    temps = (ctypes.c_float * nb)(*[float(t) for t in temperatures])
    _abi.call("hs_confidence_batched", ptrs, temps, nb, _dtype_code(x0), n, seq_len, C,
              int(x0.stride(0)), _p(row_index), _kind(kind), _reduce(reduce), _p(out["conf"]),
              _p(out.get("argmax")), _p(labels), _p(out.get("correct")), _p(ws),
              0 if ws is None else ws.numel(), _p(status), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# hs_fit_temperature (NEXT-3: Eq. 1)
# ---------------------------------------------------------------------------
T_MIN, T_MAX = 0.01831563888873418, 54.598150033144236     # e^-4, e^4: clamp range of S:112


def fit_temperature(logits: list, labels: torch.Tensor, *, n: int | None = None,
                    n_classes: int | None = None, t_lo: float = T_MIN, t_hi: float = T_MAX,
                    max_passes: int = 64, status: torch.Tensor | None = None,
                    out: dict | None = None, ws: torch.Tensor | None = None, stream=None) -> dict:
    """Fit one temperature per stage model on the same labelled validation rows
    (Eq. 1: minimise the NLL of softmax(x / T) over [t_lo, t_hi]); all stage
    models in one persistent launch.  Returns ``T`` f32[K], ``nll`` f64[K]
    (mean NLL at the last swept temperature), ``passes`` i32[K], ``used`` i64[K]."""
    import ctypes
    nb = len(logits)
    x0 = logits[0]
    _check_cuda(*logits, labels, status)
    for x in logits:
        if x.dim() != 2 or x.stride(1) != 1 or x.stride(0) != x0.stride(0) or x.dtype != x0.dtype:
            raise ValueError("stage logits must share dtype, shape and row stride")
    C = int(n_classes or x0.shape[1])
    n = int(x0.shape[0] if n is None else n)
    dev = x0.device
    out = dict(out or {})
    out.setdefault("T", torch.empty(nb, dtype=torch.float32, device=dev))
    out.setdefault("nll", torch.empty(nb, dtype=torch.float64, device=dev))
    out.setdefault("passes", torch.empty(nb, dtype=torch.int32, device=dev))
    out.setdefault("used", torch.empty(nb, dtype=torch.int64, device=dev))
    need = lib().hs_fit_temperature_workspace(nb, n)
    if ws is None or ws.numel() < need:
        ws = _temp_workspace(need, dev, stream)
    ptrs = (ctypes.c_void_p * nb)(*[x.data_ptr() for x in logits])
    _abi.call("hs_fit_temperature", ptrs, nb, _dtype_code(x0), n, C, int(x0.stride(0)), _p(labels),
              float(t_lo), float(t_hi), int(max_passes), _p(out["T"]), _p(out["nll"]),
              _p(out["passes"]), _p(out["used"]), _p(ws), ws.numel(), _p(status), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# NEXT-4: threshold performance graph (Alg. 1)
# ---------------------------------------------------------------------------
def grid_size(K: int, log2_bins: int) -> int:
    """(B+2)^(K-1) threshold vectors on the D5 grid (-1 if too many)."""
    return int(lib().hs_grid_size(int(K), int(log2_bins)))


def grid_vector(s: int, K: int, log2_bins: int) -> list:
    """Threshold indices b_0..b_{K-2} of grid vector s (b_0 most significant)."""
    import ctypes
    b = (ctypes.c_int32 * max(1, K - 1))()
    _abi.call("hs_grid_vector", int(s), int(K), int(log2_bins), b)
    return list(b)[: K - 1]


def threshold_replay(conf: torch.Tensor, correct: torch.Tensor, weights, *, log2_bins: int = 12,
                     bvecs: torch.Tensor | None = None, want_reach: bool = False,
                     out: dict | None = None, ws: torch.Tensor | None = None, stream=None) -> dict:
    """Replay the cascade for S threshold vectors (``bvecs`` [S, K-1] int32, or
    None = the whole grid): ``correct`` i64[S], ``energy`` i64[S] (sum_k reach_k
    * weights[k]), optional ``reach`` i64[S, K], ``model_correct`` i64[K]."""
    import ctypes
    _check_cuda(conf, correct, bvecs)
    K, N = int(correct.shape[0]), int(correct.shape[1])
    S = grid_size(K, log2_bins) if bvecs is None else int(bvecs.shape[0])
    dev = conf.device
    out = dict(out or {})
    out.setdefault("correct", torch.empty(S, dtype=torch.int64, device=dev))
    out.setdefault("energy", torch.empty(S, dtype=torch.int64, device=dev))
    out.setdefault("model_correct", torch.empty(K, dtype=torch.int64, device=dev))
    if want_reach:
        out.setdefault("reach", torch.empty(S, K, dtype=torch.int64, device=dev))
    need = lib().hs_threshold_replay_workspace(K, N, int(log2_bins))
    if ws is None or ws.numel() < need:
        ws = _temp_workspace(need, dev, stream)
    w = (ctypes.c_int64 * K)(*[int(x) for x in weights])
    _abi.call("hs_threshold_replay", _p(conf), _p(correct), K, N, int(log2_bins), _p(bvecs), S, w,
              _p(out["correct"]), _p(out["energy"]), _p(out.get("reach")), _p(out["model_correct"]),
              _p(ws), ws.numel(), _stream(stream))
    return out


def perf_graph(correct: torch.Tensor, energy: torch.Tensor, N: int, *, tau: int = -1, floor: int = -1,
               model_correct: torch.Tensor | None = None, K: int = 0, status: torch.Tensor | None = None,
               out: dict | None = None, ws: torch.Tensor | None = None, stream=None) -> dict:
    """Pareto frontier of the (correct, energy) points and the AP / EO picks:
    ``front_c``/``front_e``/``front_s`` i64[N+1] (first ``front_n`` valid),
    ``pick`` i64[2] = (AP vector, EO vector)."""
    _check_cuda(correct, energy, model_correct, status)
    S = int(correct.numel())
    dev = correct.device
    out = dict(out or {})
    for k in ("front_c", "front_e", "front_s"):
        out.setdefault(k, torch.empty(N + 1, dtype=torch.int64, device=dev))
    out.setdefault("front_n", torch.empty(1, dtype=torch.int64, device=dev))
    out.setdefault("pick", torch.empty(2, dtype=torch.int64, device=dev))
    need = lib().hs_perf_graph_workspace(N)
    if ws is None or ws.numel() < need:
        ws = _temp_workspace(need, dev, stream)
    _abi.call("hs_perf_graph", _p(correct), _p(energy), S, int(N), int(tau), int(floor),
              _p(model_correct), int(K), _p(out["front_c"]), _p(out["front_e"]), _p(out["front_s"]),
              _p(out["front_n"]), _p(out["pick"]), _p(ws), ws.numel(), _p(status), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# Peer-memory forwarding of deferred requests (hs_forward_*)
# ---------------------------------------------------------------------------
def _ptr_array(ptrs):
    import ctypes
    return (ctypes.c_void_p * len(ptrs))(*[int(p) if p else None for p in ptrs])


# ---------------------------------------------------------------------------
# Multi-GPU group over peer memory (hs_peer_*; dist.PeerGroup builds the group)
# ---------------------------------------------------------------------------
def peer_region_bytes(world: int, cap: int, payload_row_bytes: int = 0, log2_bins: int = 12) -> int:
    return int(lib().hs_peer_region_bytes(int(world), int(cap), int(payload_row_bytes), int(log2_bins)))


def _dest_array(dest_ranks):
    import ctypes
    if dest_ranks is None:
        return None, 0
    return (ctypes.c_int32 * len(dest_ranks))(*[int(d) for d in dest_ranks]), len(dest_ranks)


def peer_forward(g, set_: int, ids: torch.Tensor, d_count: torch.Tensor, recv_count: torch.Tensor, *,
                 payload: torch.Tensor | None = None, dest_ranks=None, status: torch.Tensor | None = None,
                 stream=None):
    """hs_peer_forward: this rank's deferred ids[:*d_count] (+ payload rows) to
    their blocks of the global stable list on ``dest_ranks`` (None = all ranks);
    this rank's block lands in receive set ``set_`` (count -> recv_count)."""
    import ctypes
    dr, nd = _dest_array(dest_ranks)
    _abi.call("hs_peer_forward", ctypes.byref(g), int(set_), _p(ids), _p(payload), _p(d_count), dr, nd,
              _p(recv_count), _p(status), _stream(stream))


def peer_forward_publish(g, d_count: torch.Tensor, status: torch.Tensor | None = None, stream=None):
    import ctypes
    _abi.call("hs_peer_forward_publish", ctypes.byref(g), _p(d_count), _p(status), _stream(stream))


def peer_forward_scatter(g, set_: int, ids: torch.Tensor, recv_count: torch.Tensor, *,
                         payload: torch.Tensor | None = None, dest_ranks=None,
                         status: torch.Tensor | None = None, stream=None):
    import ctypes
    dr, nd = _dest_array(dest_ranks)
    _abi.call("hs_peer_forward_scatter", ctypes.byref(g), int(set_), _p(ids), _p(payload), dr, nd,
              _p(recv_count), _p(status), _stream(stream))


def peer_forward_wait(g, status: torch.Tensor | None = None, stream=None):
    import ctypes
    _abi.call("hs_peer_forward_wait", ctypes.byref(g), _p(status), _stream(stream))


def calibrate_thresholds_peer(conf: torch.Tensor, correct: torch.Tensor, g, *, log2_bins: int = 12,
                              target: int = -1, out: dict | None = None, ws: torch.Tensor | None = None,
                              status: torch.Tensor | None = None, stream=None) -> dict:
    """AP calibration over a request-sharded validation set: this rank's shard
    (conf f32 [K-1, N], correct u8 [K, N]); the per-round histograms are summed
    across the group inside the calibration kernel (hs_calibrate_thresholds_peer)."""
    import ctypes
    _check_cuda(conf, correct)
    K, N = int(correct.shape[0]), int(correct.shape[1])
    dev = correct.device
    out = _calib_out(K, dev, out)
    need = lib().hs_calibrate_workspace(K, log2_bins)
    if ws is None or ws.numel() < need:
        ws = _temp_workspace(need, dev, stream)
    _abi.call("hs_calibrate_thresholds_peer", _p(conf), _p(correct), K, N, int(log2_bins), int(target),
              _p(out["b"]), _p(out["t"]), _p(out["reach"]), _p(out["handled"]), _p(out["correct_total"]),
              ctypes.byref(g), _p(ws), ws.numel(), _p(status), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# The library's NCCL communicator and request-sharded calibration (hs_comm_*)
# ---------------------------------------------------------------------------
def comm_unique_id() -> bytes:
    """A 128-byte NCCL unique id (create on rank 0, share with the group)."""
    import ctypes
    buf = ctypes.create_string_buffer(128)
    _abi.call("hs_comm_unique_id", buf)
    return bytes(buf.raw)


def comm_create(uid: bytes, rank: int, world: int, device: int) -> int:
    """Join the group (collective); returns the library-owned handle."""
    import ctypes
    h = ctypes.c_void_p()
    _abi.call("hs_comm_create", ctypes.create_string_buffer(uid, 128), int(rank), int(world),
              int(device), ctypes.byref(h))
    return int(h.value)


def comm_destroy(comm: int):
    _abi.call("hs_comm_destroy", comm)


def forward_nccl(ids: torch.Tensor, d_count: torch.Tensor, comm: int, world: int, *,
                 dest_ranks: list | None = None, payload: torch.Tensor | None = None,
                 payload_row_bytes: int = 0, recv_cap: int | None = None, out: dict | None = None,
                 ws: torch.Tensor | None = None, stream=None):
    """NCCL forwarding of this rank's deferred list (hs_forward_nccl): returns
    (recv_ids, recv_payload, n_recv) with n_recv read back to the host."""
    import ctypes
    dev = ids.device
    dest = list(range(world)) if dest_ranks is None else list(dest_ranks)
    cap = int(recv_cap if recv_cap is not None else world * ids.numel())
    out = dict(out or {})
    out.setdefault("recv_ids", torch.empty(max(cap, 1), dtype=torch.int64, device=dev))
    if payload_row_bytes:
        out.setdefault("recv_payload", torch.empty(max(cap, 1) * payload_row_bytes, dtype=torch.uint8, device=dev))
    need = lib().hs_forward_nccl_workspace(world)
    if ws is None or ws.numel() < need:
        ws = _temp_workspace(need, dev, stream)
    dr = (ctypes.c_int32 * len(dest))(*dest)
    n = ctypes.c_int64()
    _abi.call("hs_forward_nccl", _p(ids), _p(payload), int(payload_row_bytes), _p(d_count), dr, len(dest),
              _p(out["recv_ids"]), _p(out.get("recv_payload")), cap, ctypes.byref(n), comm, _p(ws),
              ws.numel(), _stream(stream))
    return out["recv_ids"][: n.value], (out["recv_payload"][: n.value * payload_row_bytes]
                                         if payload_row_bytes else None), n.value


def calibrate_thresholds_comm(conf: torch.Tensor, correct: torch.Tensor, comm: int | None, *,
                              log2_bins: int = 12, target: int = -1, refine_passes: int = 0,
                              out: dict | None = None, ws: torch.Tensor | None = None,
                              stream=None) -> dict:
    """hs_calibrate_thresholds over a validation set sharded across the ranks
    of ``comm`` (this rank's shard in conf / correct); identical b_k on every
    rank (hs_calibrate_thresholds_comm_ex; refinement passes summed across ranks)."""
    _check_cuda(conf, correct)
    K, N = int(correct.shape[0]), int(correct.shape[1])
    out = _calib_out(K, conf.device, out)
    if ws is None:
        ws = calibrate_workspace(K, log2_bins, conf.device)
    _abi.call("hs_calibrate_thresholds_comm_ex", _p(conf), _p(correct), K, N, int(log2_bins), int(target),
              int(refine_passes), _p(out["b"]), _p(out["t"]), _p(out["reach"]), _p(out["handled"]),
              _p(out["correct_total"]), comm, _p(ws), ws.numel(), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# hs_route_compact
# ---------------------------------------------------------------------------
def route_compact(conf: torch.Tensor, threshold: float | torch.Tensor, *, is_last: bool = False,
                  n: int | None = None, d_n: torch.Tensor | None = None,
                  ids: torch.Tensor | None = None, pred: torch.Tensor | None = None,
                  pred_len: int = 1, payload: torch.Tensor | None = None,
                  out: dict | None = None, ws: torch.Tensor | None = None, stream=None) -> dict:
    """Threshold test + stable split.  Returns capacity-sized
    buffers and ``counts`` (device int64[2] = {#accepted, #deferred})."""
    _check_cuda(conf, d_n, ids, pred, payload)
    n = int(conf.numel() if n is None else n)
    dev = conf.device
    out = dict(out or {})
    if "acc_ids" not in out:
        out["acc_ids"] = torch.empty(n, dtype=torch.int64, device=dev)
    if "acc_conf" not in out:
        out["acc_conf"] = torch.empty(n, dtype=torch.float32, device=dev)
    if pred is not None:
        if "acc_pred" not in out:
            out["acc_pred"] = torch.empty(n * pred_len, dtype=torch.int32, device=dev)
    if "def_ids" not in out:
        out["def_ids"] = torch.empty(n, dtype=torch.int64, device=dev)
    if "def_pos" not in out:
        out["def_pos"] = torch.empty(n, dtype=torch.int64, device=dev)
    P = 0
    if payload is not None:
        P = payload.element_size()
        for d in payload.shape[1:]:
            P *= int(d)
        if "def_payload" not in out:
            out["def_payload"] = torch.empty_like(payload)
    if "counts" not in out:
        out["counts"] = torch.zeros(2, dtype=torch.int64, device=dev)
    need = lib().hs_route_compact_workspace(n)
    if ws is None:
        ws = workspace(need, dev)
    d_thr = threshold if isinstance(threshold, torch.Tensor) else None
    thr = 0.0 if d_thr is not None else float(threshold)
    _abi.call("hs_route_compact", _p(conf), n, _p(d_n), thr, _p(d_thr), int(bool(is_last)),
              _p(ids), _p(pred), int(pred_len), _p(out["acc_ids"]), _p(out["acc_conf"]),
              _p(out.get("acc_pred")), _p(out["def_ids"]), _p(out["def_pos"]), _p(payload), P,
              _p(out.get("def_payload")), _p(out["counts"]), _p(ws), ws.numel(), _stream(stream))
    return out


# ---------------------------------------------------------------------------
# hs_cascade_step
# ---------------------------------------------------------------------------
def cascade_step(stage: int, n_stages: int, logits: torch.Tensor, threshold, *, n: int,
                 seq_len: int = 1, n_classes: int | None = None, temperature: float = 1.0,
                 kind="maxprob", reduce="none", row_index: torch.Tensor | None = None,
                 d_n: torch.Tensor | None = None, ids: torch.Tensor | None = None,
                 payload: torch.Tensor | None = None, payload_row_bytes: int = 0,
                 out: dict | None = None, ws: torch.Tensor | None = None,
                 status: torch.Tensor | None = None, overlap_previous: bool = False,
                 top_k: int = 0, peer=None, peer_set: int = 0, next_ranks=None,
                 recv_count: torch.Tensor | None = None, stream=None) -> dict:
    """One model m_k of the cascade: confidence -> threshold -> compaction/gather.

    ``peer`` (a dist.PeerGroup's ``g``): hs_cascade_step_peer -- the deferred
    list is then forwarded to ``next_ranks`` (None = all ranks) into receive
    set ``peer_set`` of the group (count -> ``recv_count``).

    ``overlap_previous`` (HS_STEP_OVERLAP_PREVIOUS): the confidence kernel runs
    next to the previous libhs kernel on the stream; the caller guarantees that
    kernel does not touch this step's inputs or workspace."""
    _check_cuda(logits, row_index, d_n, ids, payload, status)
    if row_index is None and d_n is None and logits.shape[0] < n * seq_len:
        raise ValueError(f"cascade_step: {n} items x {seq_len} tokens but logits has {logits.shape[0]} rows")
    C = int(n_classes or logits.shape[1])
    dev = logits.device
    out = dict(out or {})
    if "acc_ids" not in out:
        out["acc_ids"] = torch.empty(n, dtype=torch.int64, device=dev)
    if "acc_conf" not in out:
        out["acc_conf"] = torch.empty(n, dtype=torch.float32, device=dev)
    if "acc_pred" not in out:
        out["acc_pred"] = torch.empty(n * seq_len, dtype=torch.int32, device=dev)
    if "next_ids" not in out:
        out["next_ids"] = torch.empty(n, dtype=torch.int64, device=dev)
    if payload is not None and payload_row_bytes > 0:
        if "next_payload" not in out:
            out["next_payload"] = torch.empty(n * payload_row_bytes, dtype=torch.uint8, device=dev)
    if "counts" not in out:
        out["counts"] = torch.zeros(2, dtype=torch.int64, device=dev)
    need = lib().hs_cascade_step_workspace(n, seq_len)
    if ws is None:
        ws = workspace(need, dev)
    d_thr = threshold if isinstance(threshold, torch.Tensor) else None
    thr = 0.0 if d_thr is not None else float(threshold)
    flags = (HS_STEP_OVERLAP_PREVIOUS if overlap_previous else 0) | _rows_capacity_flag(logits, n * seq_len, row_index)
    if peer is not None:
        import ctypes
        dr, nd = _dest_array(next_ranks)
        _abi.call("hs_cascade_step_peer", int(stage), int(n_stages), _p(logits), _dtype_code(logits),
                  int(n), int(seq_len), C, int(logits.stride(0)), _p(row_index), _p(d_n),
                  float(temperature), _kind(kind), _reduce(reduce), thr, _p(d_thr), _p(ids), _p(payload),
                  int(payload_row_bytes), _p(out["acc_ids"]), _p(out["acc_conf"]), _p(out["acc_pred"]),
                  _p(out["next_ids"]), _p(out.get("next_payload")), _p(out["counts"]), _p(ws),
                  ws.numel(), _p(status), int(top_k), flags,
                  ctypes.byref(peer), int(peer_set), dr, nd, _p(recv_count), _stream(stream))
        return out
    _abi.call("hs_cascade_step_ex", int(stage), int(n_stages), _p(logits), _dtype_code(logits),
              int(n), int(seq_len), C, int(logits.stride(0)), _p(row_index), _p(d_n),
              float(temperature), _kind(kind), _reduce(reduce), thr, _p(d_thr), _p(ids), _p(payload),
              int(payload_row_bytes), _p(out["acc_ids"]), _p(out["acc_conf"]), _p(out["acc_pred"]),
              _p(out["next_ids"]), _p(out.get("next_payload")), _p(out["counts"]), _p(ws),
              ws.numel(), _p(status), int(top_k), flags, _stream(stream))
    return out


# ---------------------------------------------------------------------------
# hs_calibrate_*
# ---------------------------------------------------------------------------
def _calib_out(K: int, dev, out: dict | None):
    out = dict(out or {})
    if "b" not in out:
        out["b"] = torch.empty(K - 1, dtype=torch.int32, device=dev)
    if "t" not in out:
        out["t"] = torch.empty(K, dtype=torch.float32, device=dev)
    if "reach" not in out:
        out["reach"] = torch.empty(K, dtype=torch.int64, device=dev)
    if "handled" not in out:
        out["handled"] = torch.empty(K, dtype=torch.int64, device=dev)
    if "correct_total" not in out:
        out["correct_total"] = torch.empty(1, dtype=torch.int64, device=dev)
    return out


def calibrate_thresholds(conf: torch.Tensor, correct: torch.Tensor, *, log2_bins: int = 12,
                         target: int = -1, refine_passes: int = 0, out: dict | None = None,
                         ws: torch.Tensor | None = None, stream=None) -> dict:
    """AP threshold calibration on the validation set.
    conf: f32 [K-1, N]; correct: u8 [K, N]."""
    _check_cuda(conf, correct)
    K, N = int(correct.shape[0]), int(correct.shape[1])
    if conf.dtype != torch.float32 or correct.dtype != torch.uint8:
        raise TypeError("conf must be float32 and correct uint8")
    if tuple(conf.shape) != (K - 1, N) or not conf.is_contiguous() or not correct.is_contiguous():
        raise ValueError("conf must be contiguous [K-1, N], correct contiguous [K, N]")
    dev = conf.device
    out = _calib_out(K, dev, out)
    need = lib().hs_calibrate_workspace(K, log2_bins)
    if ws is None or ws.numel() < need:
        ws = _temp_workspace(need, dev, stream)
    _abi.call("hs_calibrate_thresholds", _p(conf), _p(correct), K, N, int(log2_bins), int(target),
              int(refine_passes), _p(out["b"]), _p(out["t"]), _p(out["reach"]),
              _p(out["handled"]), _p(out["correct_total"]), _p(ws), ws.numel(), _stream(stream))
    return out


def calibrate_begin(K: int, log2_bins: int, target: int, ws: torch.Tensor, stream=None):
    _abi.call("hs_calibrate_begin", int(K), int(log2_bins), int(target), _p(ws), ws.numel(),
              _stream(stream))


def calibrate_hist_view(ws: torch.Tensor, log2_bins: int) -> torch.Tensor:
    """The int32 [3, B+2] histogram inside a calibration workspace (for all-reduce)."""
    off = lib().hs_calibrate_hist_ptr(ws.data_ptr()) - ws.data_ptr()
    nb = (1 << log2_bins) + 2
    return ws[off: off + 3 * nb * 4].view(torch.int32).view(3, nb)


def calibrate_histogram(conf, correct, round_: int, b: torch.Tensor, *, log2_bins: int,
                        ws: torch.Tensor, stream=None):
    K, N = int(correct.shape[0]), int(correct.shape[1])
    _abi.call("hs_calibrate_histogram", _p(conf), _p(correct), K, N, int(log2_bins), int(round_),
              _p(b), _p(ws), ws.numel(), _stream(stream))


def calibrate_select(K: int, round_: int, out: dict, *, log2_bins: int, ws: torch.Tensor,
                     stream=None):
    _abi.call("hs_calibrate_select", int(K), int(log2_bins), int(round_), _p(out["b"]),
              _p(out["t"]), _p(out["reach"]), _p(out["handled"]), _p(out["correct_total"]),
              _p(ws), ws.numel(), _stream(stream))


def calibrate_workspace(K: int, log2_bins: int, device) -> torch.Tensor:
    return torch.empty(max(lib().hs_calibrate_workspace(K, log2_bins), 16), dtype=torch.uint8,
                       device=device)


# ---------------------------------------------------------------------------
# A K-stage cascade with preallocated buffers (no host round trip between
# stages: each stage's batch size and threshold are read on the device).
# ---------------------------------------------------------------------------
@dataclasses.dataclass
class StageSpec:
    n_classes: int
    temperature: float = 1.0
    seq_len: int = 1
    kind: int = MAXPROB
    reduce: int = SEQ_NONE
    top_k: int = 0          # NEXT-2: restricted softmax over the top_k logits (0 = full)


class Cascade:
    """Routes a batch through models m_1..m_K.

    ``route(logits, thresholds)``: logits[k] holds stage k's logits for every
    request id (row = id, ``by_id=True``) or for stage k's batch in order
    (``by_id=False``); thresholds is a device f32[K] (e.g. from
    ``calibrate_thresholds``) or a list of floats.  All stages are launched
    stream-ordered without host synchronisation; results stay on the device:
    ``acc_ids[k][:counts[k,0]]``, ``acc_pred[k]``, ``acc_conf[k]``.
    """

    def __init__(self, n_cap: int, stages: list[StageSpec], device, payload_row_bytes: int = 0):
        self.n_cap = int(n_cap)
        self.stages = stages
        self.K = len(stages)
        self.device = torch.device(device)
        self.P = int(payload_row_bytes)
        L = max(s.seq_len for s in stages)
        dev = self.device
        self.counts = torch.zeros(self.K, 2, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)
        self.outs = []
        for k, s in enumerate(stages):
            o = {"acc_ids": torch.empty(n_cap, dtype=torch.int64, device=dev),
                 "acc_conf": torch.empty(n_cap, dtype=torch.float32, device=dev),
                 "acc_pred": torch.empty(n_cap * s.seq_len, dtype=torch.int32, device=dev),
                 "next_ids": torch.empty(n_cap, dtype=torch.int64, device=dev),
                 "counts": self.counts[k]}
            if self.P and k < self.K - 1:
                o["next_payload"] = torch.empty(n_cap * self.P, dtype=torch.uint8, device=dev)
            self.outs.append(o)
        self.ws = workspace(lib().hs_cascade_step_workspace(n_cap, L), dev)

    def route(self, logits: list, thresholds, *, n: int | None = None, ids=None, payload=None,
              by_id: bool = True, overlap_first: bool = False, peer=None, next_ranks=None,
              events=None, upto: int | None = None, split: bool = False, stream=None):
        """Run the K stages.  ``overlap_first``: stage 1's confidence kernel runs
        next to the previous libhs kernel (e.g. the calibration it does not
        depend on); see hs_cascade_step_ex / HS_STEP_OVERLAP_PREVIOUS.

        ``peer`` (a dist.PeerGroup): request-sharded cascade over a group of
        GPUs -- after every stage the deferred list is forwarded over peer
        memory (hs_cascade_step_peer) to ``next_ranks[k]`` (None = all ranks:
        the balanced placement), and stage k+1 routes the block this rank
        received (receive set k % 2, count ``peer.recv_count[k]``).  With
        ``by_id`` the stage logits are indexed by request id; otherwise they are
        the dense batch of the block this rank receives.

        ``events`` (timing): a list of 2K CUDA events; events[2k] is recorded
        before stage k and events[2k+1] between its compaction and its forward
        (the forward is then launched as its own call, same kernels).
        ``upto``: run stages 0..upto only (and their forwards).
        ``split``: single GPU, dense stage batches (``by_id=False``): each
        stage's confidence also counts its deferred items
        (hs_cascade_confidence), the next stage's confidence starts from that
        count, and every compaction (hs_cascade_compact) runs on a side stream
        off the critical path (joined before returning)."""
        if split and peer is None and not by_id and events is None:
            return self._route_split(logits, thresholds, n=n, ids=ids, payload=payload,
                                     overlap_first=overlap_first, upto=upto, stream=stream)
        n = self.n_cap if n is None else int(n)
        d_thr = thresholds if isinstance(thresholds, torch.Tensor) else None
        for k, s in enumerate(self.stages):
            if upto is not None and k > upto:
                break
            prev = self.outs[k - 1] if k else None
            if k and peer is not None:
                cur_ids = peer.recv_ids((k - 1) % 2)
                cur_payload = peer.recv_payload((k - 1) % 2) if self.P else None
                d_n = peer.recv_count[k - 1: k]
            else:
                cur_ids = prev["next_ids"] if k else ids
                cur_payload = prev.get("next_payload") if k else payload
                d_n = prev["counts"][1:2] if k else None
            thr = d_thr[k:k + 1] if d_thr is not None else float(thresholds[k] if k < self.K - 1 else 0.0)
            row_index = cur_ids if by_id else None
            if by_id and cur_ids is None:
                row_index = None   # stage 1 with identity ids: row = id = position
            # stages after the first: capacity-sized (a placed rank may receive
            # more than its own shard), the live count comes from d_n
            nk = n if (k == 0 or peer is None) else self.n_cap
            kw = {}
            fwd = peer is not None and k < self.K - 1
            if fwd and events is None:
                kw = {"peer": peer.g, "peer_set": k % 2, "recv_count": peer.recv_count[k:k + 1],
                      "next_ranks": None if next_ranks is None else next_ranks[k]}
            if events is not None:
                events[2 * k].record(stream)
            cascade_step(k, self.K, logits[k], thr, n=nk, seq_len=s.seq_len, n_classes=s.n_classes,
                         temperature=s.temperature, kind=s.kind, reduce=s.reduce,
                         row_index=row_index, d_n=d_n,
                         ids=cur_ids, payload=cur_payload, payload_row_bytes=self.P,
                         out=self.outs[k], ws=self.ws, status=self.status,
                         overlap_previous=overlap_first and k == 0, top_k=s.top_k,
                         stream=stream, **kw)
            if events is not None:
                events[2 * k + 1].record(stream)
                if fwd:
                    peer_forward(peer.g, k % 2, self.outs[k]["next_ids"], self.outs[k]["counts"][1:2],
                                 peer.recv_count[k:k + 1], payload=self.outs[k].get("next_payload"),
                                 dest_ranks=None if next_ranks is None else next_ranks[k],
                                 status=peer.status, stream=stream)
        return self

    def _route_split(self, logits, thresholds, *, n, ids, payload, overlap_first, upto, stream):
        import ctypes
        n = self.n_cap if n is None else int(n)
        main = stream if stream is not None else torch.cuda.current_stream(self.device)
        if not hasattr(self, "_side"):
            L = max(s.seq_len for s in self.stages)
            self._side = torch.cuda.Stream(device=self.device)
            self._stage_ws = [workspace(lib().hs_cascade_step_workspace(self.n_cap, L), self.device)
                              for _ in range(self.K)]
            self._defer = torch.zeros(self.K, dtype=torch.int64, device=self.device)
            self._ev = [torch.cuda.Event() for _ in range(self.K)]
        d_thr = thresholds if isinstance(thresholds, torch.Tensor) else None
        side = self._side
        with torch.cuda.stream(main):
            self._defer.zero_()
        for k, s in enumerate(self.stages):
            if upto is not None and k > upto:
                break
            thr = d_thr[k:k + 1] if d_thr is not None else float(thresholds[k] if k < self.K - 1 else 0.0)
            dt, th = (_p(thr), 0.0) if isinstance(thr, torch.Tensor) else (None, float(thr))
            d_n = self._defer[k - 1:k] if k else None
            x = logits[k]
            ws = self._stage_ws[k]
            last = k == self.K - 1
            _abi.call("hs_cascade_confidence", k, self.K, _p(x), _dtype_code(x), n, int(s.seq_len),
                      int(s.n_classes), int(x.stride(0)), None, _p(d_n), float(s.temperature),
                      _kind(s.kind), _reduce(s.reduce), th, dt,
                      None if last else _p(self._defer[k:k + 1]), _p(ws), ws.numel(), _p(self.status),
                      int(s.top_k), HS_STEP_OVERLAP_PREVIOUS if (overlap_first and k == 0) else 0,
                      main.cuda_stream)
            self._ev[k].record(main)
            side.wait_event(self._ev[k])
            prev = self.outs[k - 1] if k else None
            o = self.outs[k]
            _abi.call("hs_cascade_compact", k, self.K, n, int(s.seq_len), _p(d_n), th, dt,
                      _p(prev["next_ids"] if k else ids),
                      _p(prev.get("next_payload") if k else payload), self.P,
                      _p(o["acc_ids"]), _p(o["acc_conf"]), _p(o["acc_pred"]), _p(o["next_ids"]),
                      _p(o.get("next_payload")), _p(o["counts"]), _p(ws), ws.numel(), side.cuda_stream)
        main.wait_stream(side)
        return self

    def results(self):
        """Host copy of the per-stage accepted lists (synchronises)."""
        counts = self.counts.cpu()
        res = []
        for k, s in enumerate(self.stages):
            na = int(counts[k, 0])
            o = self.outs[k]
            res.append({"ids": o["acc_ids"][:na].cpu(), "conf": o["acc_conf"][:na].cpu(),
                        "pred": o["acc_pred"][:na * s.seq_len].cpu(), "n_acc": na,
                        "n_def": int(counts[k, 1])})
        return res


# ---------------------------------------------------------------------------
# Skip connections (NEXT-1): hs_skip_select / hs_skip_route
# ---------------------------------------------------------------------------
SKIP_UNIFORM, SKIP_DECADE = 0, 1


def skip_edges(threshold: float, successors: int, mode: int = SKIP_UNIFORM) -> list:
    """fp32 band edges inside [0, t) (host helper, hs_skip_edges)."""
    import ctypes
    n = max(successors - 1, 0)
    buf = (ctypes.c_float * max(n, 1))()
    _abi.call("hs_skip_edges", float(threshold), int(successors), int(mode), ctypes.addressof(buf))
    return [buf[i] for i in range(n)]


def skip_select(dest: torch.Tensor, stage: int, *, out: dict | None = None,
                ws: torch.Tensor | None = None, stream=None) -> dict:
    """Batch of model `stage`: requests r with dest[r] == stage, increasing r."""
    _check_cuda(dest)
    n = int(dest.numel())
    out = dict(out or {})
    if "ids" not in out:
        out["ids"] = torch.empty(max(n, 1), dtype=torch.int64, device=dest.device)
    if "counts" not in out:
        out["counts"] = torch.zeros(2, dtype=torch.int64, device=dest.device)
    if ws is None:
        ws = workspace(lib().hs_route_compact_workspace(n), dest.device)
    _abi.call("hs_skip_select", _p(dest), n, int(stage), _p(out["ids"]), _p(out["counts"]), _p(ws),
              ws.numel(), _stream(stream))
    return out


def skip_route(conf: torch.Tensor, threshold, stage: int, n_stages: int, dest: torch.Tensor,
               ids: torch.Tensor, *, mode: int = SKIP_UNIFORM, n: int | None = None,
               d_n: torch.Tensor | None = None, pred: torch.Tensor | None = None,
               pred_len: int = 1, out: dict | None = None, ws: torch.Tensor | None = None,
               stream=None) -> dict:
    """Threshold test of model `stage`'s batch with skip bands; updates dest."""
    _check_cuda(conf, dest, ids, d_n, pred)
    n = int(conf.numel() if n is None else n)
    dev = conf.device
    out = dict(out or {})
    if "acc_ids" not in out:
        out["acc_ids"] = torch.empty(max(n, 1), dtype=torch.int64, device=dev)
    if "acc_conf" not in out:
        out["acc_conf"] = torch.empty(max(n, 1), dtype=torch.float32, device=dev)
    if pred is not None and "acc_pred" not in out:
        out["acc_pred"] = torch.empty(max(n, 1) * pred_len, dtype=torch.int32, device=dev)
    if "counts" not in out:
        out["counts"] = torch.zeros(2, dtype=torch.int64, device=dev)
    if ws is None:
        ws = workspace(lib().hs_route_compact_workspace(n), dev)
    d_thr = threshold if isinstance(threshold, torch.Tensor) else None
    thr = 0.0 if d_thr is not None else float(threshold)
    _abi.call("hs_skip_route", _p(conf), n, _p(d_n), thr, _p(d_thr), int(stage), int(n_stages),
              int(mode), _p(ids), _p(pred), int(pred_len), _p(out["acc_ids"]), _p(out["acc_conf"]),
              _p(out.get("acc_pred")), _p(dest), _p(out["counts"]), _p(ws), ws.numel(),
              _stream(stream))
    return out


class SkipCascade:
    """The cascade with skip connections: per model k, select its batch from the
    per-request `dest` array (hs_skip_select), compute the confidences of those
    rows (hs_confidence, logits indexed by request id), then threshold + band
    routing (hs_skip_route).  No host round trip; `dest[r] - K` is the model
    that answered request r when all stages ran."""

    def __init__(self, n_req: int, stages: list[StageSpec], device, mode: int = SKIP_UNIFORM):
        self.n = int(n_req)
        self.stages = stages
        self.K = len(stages)
        self.mode = int(mode)
        dev = torch.device(device)
        self.device = dev
        L = max(s.seq_len for s in stages)
        self.dest = torch.zeros(self.n, dtype=torch.int32, device=dev)
        self.counts = torch.zeros(self.K, 2, dtype=torch.int64, device=dev)
        self.sel_counts = torch.zeros(self.K, 2, dtype=torch.int64, device=dev)
        self.batch = [torch.empty(self.n, dtype=torch.int64, device=dev) for _ in range(self.K)]
        self.conf = torch.empty(self.n, dtype=torch.float32, device=dev)
        self.argmax = torch.empty(self.n * L, dtype=torch.int32, device=dev)
        self.outs = [{"acc_ids": torch.empty(self.n, dtype=torch.int64, device=dev),
                      "acc_conf": torch.empty(self.n, dtype=torch.float32, device=dev),
                      "acc_pred": torch.empty(self.n * s.seq_len, dtype=torch.int32, device=dev),
                      "counts": self.counts[k]} for k, s in enumerate(stages)]
        self.ws_sel = workspace(lib().hs_route_compact_workspace(self.n), dev)
        self.ws_route = workspace(lib().hs_route_compact_workspace(self.n), dev)
        self.ws_conf = torch.empty(max(16, self.n * L * 5 + 1024), dtype=torch.uint8, device=dev)
        self.ids0 = torch.arange(self.n, dtype=torch.int64, device=dev)
        self.status = torch.zeros(1, dtype=torch.int32, device=dev)

    def route(self, logits: list, thresholds, stream=None):
        d_thr = thresholds if isinstance(thresholds, torch.Tensor) else None
        self.dest.zero_()
        for k, s in enumerate(self.stages):
            if k == 0:
                ids, d_n = self.ids0, None
            else:
                skip_select(self.dest, k, out={"ids": self.batch[k], "counts": self.sel_counts[k]},
                            ws=self.ws_sel, stream=stream)
                ids, d_n = self.batch[k], self.sel_counts[k][1:2]
            confidence(logits[k], n=self.n, seq_len=s.seq_len, n_classes=s.n_classes,
                       temperature=s.temperature, kind=s.kind, reduce=s.reduce, row_index=ids,
                       d_n=d_n, out={"conf": self.conf, "argmax": self.argmax}, ws=self.ws_conf,
                       status=self.status, stream=stream)
            thr = d_thr[k:k + 1] if d_thr is not None else float(thresholds[k] if k < self.K - 1 else 0.0)
            skip_route(self.conf, thr, k, self.K, self.dest, ids, mode=self.mode, n=self.n, d_n=d_n,
                       pred=self.argmax, pred_len=s.seq_len, out=self.outs[k], ws=self.ws_route,
                       stream=stream)
        return self

    def results(self):
        counts = self.counts.cpu()
        sel = self.sel_counts.cpu()
        res = []
        for k, s in enumerate(self.stages):
            na = int(counts[k, 0])
            nb = self.n if k == 0 else int(sel[k, 1])
            res.append({"ids": self.outs[k]["acc_ids"][:na].cpu(),
                        "batch": (self.ids0 if k == 0 else self.batch[k])[:nb].cpu(),
                        "pred": self.outs[k]["acc_pred"][:na * s.seq_len].cpu(), "n_acc": na})
        return res
