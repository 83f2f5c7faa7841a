"""CPU oracle for the HybridServe cascade router -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline``
/ ``--impl reference`` legs may import this package.  The product package
``paper_2505_12566_b200`` never imports it; the two share no code.

The arithmetic lives in ``hs_oracle.c`` (plain C, fp64, Neumaier sums); this
module only marshals numpy arrays into it and derives the per-stage lists of
the cascade statement with ``numpy.flatnonzero``.  Citations are
PAPER.md line numbers (``P:<n>``); readings are listed in DESIGN.md.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hs_oracle.c")
_LIB = os.path.join(_HERE, "libhs_oracle.so")
_lock = threading.Lock()
_lib = None

F32, BF16 = 0, 1
MAXPROB, MAXPROB_SQ, ENTROPY = 0, 1, 2
SEQ_NONE, SEQ_MIN, SEQ_MEAN = 0, 1, 2

_P = ctypes.c_void_p
_I64 = ctypes.c_int64


def build(force: bool = False) -> str:
    """Compile hs_oracle.c with gcc (plain -O2, IEEE semantics, no fast-math)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-o", tmp, _SRC,
                               "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


def lib():
    global _lib
    with _lock:
        if _lib is None:
            L = ctypes.CDLL(build())
            L.hso_row_stats.argtypes = [_P, _I64, ctypes.c_double, _P, _P, _P]
            L.hso_row_stats.restype = ctypes.c_int
            L.hso_confidence.argtypes = [_P, ctypes.c_int, _I64, ctypes.c_int, _I64, _I64, _P,
                                         ctypes.c_double, ctypes.c_int, ctypes.c_int, _I64,
                                         _P, _P, _P, _P, _P, ctypes.c_int]
            L.hso_row_stats_topk.argtypes = [_P, _I64, ctypes.c_double, _I64, _P, _P, _P]
            L.hso_row_stats_topk.restype = ctypes.c_int
            L.hso_confidence.restype = ctypes.c_int
            L.hso_route.argtypes = [_P, _I64, ctypes.c_double, ctypes.c_int, _P, _P, _P, _P]
            L.hso_route.restype = None
            L.hso_cascade.argtypes = [ctypes.c_int, _I64, _P, _P, _P]
            L.hso_cascade.restype = None
            L.hso_calibrate.argtypes = [ctypes.c_int, _I64, _P, _P, ctypes.c_int, _I64,
                                        ctypes.c_int, _P, _P, _P, _P, _P]
            L.hso_calibrate.restype = ctypes.c_int
            L.hso_nll.argtypes = [_P, ctypes.c_int, _I64, _I64, _I64, _P, ctypes.c_double, _P]
            L.hso_nll.restype = ctypes.c_double
            L.hso_fit_temperature.argtypes = [_P, ctypes.c_int, _I64, _I64, _I64, _P,
                                              ctypes.c_double, ctypes.c_double]
            L.hso_fit_temperature.restype = ctypes.c_double
            L.hso_replay.argtypes = [ctypes.c_int, _I64, _P, _P, ctypes.c_int, _I64, _P, _P, _P,
                                     _P, _P]
            L.hso_replay.restype = None
            L.hso_skip_edges.argtypes = [ctypes.c_double, ctypes.c_int, ctypes.c_int, _P]
            L.hso_skip_edges.restype = None
            L.hso_skip_band.argtypes = [ctypes.c_double, _P, ctypes.c_int]
            L.hso_skip_band.restype = ctypes.c_int
            L.hso_cascade_skip.argtypes = [ctypes.c_int, _I64, _P, _P, ctypes.c_int, _P, _P]
            L.hso_cascade_skip.restype = None
            _lib = L
    return _lib


def _ptr(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def default_threads() -> int:
    return max(1, os.cpu_count() or 1)


# --------------------------------------------------------------------------
# D1: one row.  P:373-391 (temperature-scaled softmax).
# --------------------------------------------------------------------------
def row_stats(x, T: float = 1.0, top_k: int = 0):
    """(p_max, H [nats], argmax) of one logits row in fp64; None if invalid.
    top_k > 0: statistics of the softmax restricted to the K largest logits
    (NEXT-2, reading G4)."""
    x = np.ascontiguousarray(np.asarray(x, dtype=np.float64))
    p = ctypes.c_double()
    h = ctypes.c_double()
    a = ctypes.c_int64()
    if top_k:
        rc = lib().hso_row_stats_topk(_ptr(x), x.size, float(T), int(top_k), ctypes.byref(p),
                                      ctypes.byref(h), ctypes.byref(a))
        return None if rc != 0 else (p.value, h.value, a.value)
    rc = lib().hso_row_stats(_ptr(x), x.size, float(T), ctypes.byref(p), ctypes.byref(h),
                             ctypes.byref(a))
    if rc != 0:
        return None
    return p.value, h.value, a.value


# --------------------------------------------------------------------------
# D1 + D2 batched.  P:413-430.
# --------------------------------------------------------------------------
def confidence(logits: np.ndarray, n_seq: int, seq_len: int, n_classes: int, row_stride: int,
               temperature: float, kind: int = MAXPROB, reduce: int = SEQ_NONE,
               row_index=None, labels=None, nthreads: int | None = None, top_k: int = 0):
    """Per-item confidence of a batch of logits rows.

    ``logits``: a flat float32 array, or a uint16 array of raw bf16 bits.
    Returns dict(conf f64[n], argmax i32[n*L], correct u8[n] or None, bad u8[n]).
    """
    flat = np.ascontiguousarray(logits).reshape(-1)
    if flat.dtype == np.float32:
        dtype = F32
    elif flat.dtype == np.uint16:
        dtype = BF16
    else:
        raise TypeError("oracle takes float32 or raw-bf16 (uint16) logits")
    n_seq = int(n_seq)
    conf = np.empty(n_seq, np.float64)
    argmax = np.empty(n_seq * seq_len, np.int32)
    bad = np.empty(n_seq, np.uint8)
    ri = None if row_index is None else np.ascontiguousarray(row_index, dtype=np.int64)
    lab = None if labels is None else np.ascontiguousarray(labels, dtype=np.int32)
    correct = np.empty(n_seq, np.uint8) if lab is not None else None
    rc = lib().hso_confidence(_ptr(flat), dtype, n_seq, int(seq_len), int(n_classes),
                              int(row_stride), _ptr(ri), float(temperature), int(kind),
                              int(reduce), int(top_k), _ptr(conf), _ptr(argmax), _ptr(lab), _ptr(correct),
                              _ptr(bad), int(nthreads or default_threads()))
    if rc != 0:
        raise ValueError("oracle: invalid argument")
    return {"conf": conf, "argmax": argmax, "correct": correct, "bad": bad}


# --------------------------------------------------------------------------
# D3/D4.  P:443-444.
# --------------------------------------------------------------------------
def route(conf: np.ndarray, threshold: float, is_last: bool):
    """Stable split of one stage's batch: (accepted positions, deferred positions)."""
    c = np.ascontiguousarray(conf, dtype=np.float64)
    n = c.size
    acc = np.empty(n, np.int64)
    dfr = np.empty(n, np.int64)
    na = ctypes.c_int64()
    nd = ctypes.c_int64()
    lib().hso_route(_ptr(c), n, float(threshold), int(bool(is_last)), _ptr(acc),
                    ctypes.byref(na), _ptr(dfr), ctypes.byref(nd))
    return acc[: na.value].copy(), dfr[: nd.value].copy()


def cascade(conf_by_stage: np.ndarray, thresholds) -> np.ndarray:
    """stage(r) for every request: conf_by_stage[k, r]; thresholds t[0..K-1]."""
    c = np.ascontiguousarray(conf_by_stage, dtype=np.float64)
    K, n = c.shape
    t = np.ascontiguousarray(np.asarray(thresholds, dtype=np.float64).reshape(-1)[:K])
    if t.size < K:
        t = np.concatenate([t, np.zeros(K - t.size)])
    out = np.empty(n, np.int32)
    lib().hso_cascade(int(K), int(n), _ptr(c), _ptr(t), _ptr(out))
    return out


# --------------------------------------------------------------------------
# NEXT-3: temperature fitting, Eq. 1; clamp range S:112.
# --------------------------------------------------------------------------
T_MIN, T_MAX = float(np.exp(-4.0)), float(np.exp(4.0))


def _rows(logits):
    flat = np.ascontiguousarray(logits)
    if flat.dtype == np.float32:
        return flat, F32
    if flat.dtype == np.uint16:
        return flat, BF16
    raise TypeError("oracle takes float32 or raw-bf16 (uint16) logits")


def nll(logits, labels, T: float, n_classes: int | None = None, row_stride: int | None = None):
    """(mean NLL of the temperature-scaled softmax, rows used) in fp64."""
    x, dt = _rows(logits)
    n = x.shape[0]
    C = int(n_classes or x.shape[1])
    stride = int(row_stride or x.shape[1])
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    used = ctypes.c_int64()
    v = lib().hso_nll(_ptr(x), dt, n, C, stride, _ptr(lab), float(T), ctypes.byref(used))
    return v, used.value


def fit_temperature(logits, labels, n_classes: int | None = None, row_stride: int | None = None,
                    t_lo: float = T_MIN, t_hi: float = T_MAX) -> float:
    """argmin_T NLL(T) over [t_lo, t_hi] (bisection on the beta-derivative)."""
    x, dt = _rows(logits)
    n = x.shape[0]
    C = int(n_classes or x.shape[1])
    stride = int(row_stride or x.shape[1])
    lab = np.ascontiguousarray(labels, dtype=np.int32)
    return lib().hso_fit_temperature(_ptr(x), dt, n, C, stride, _ptr(lab), float(t_lo), float(t_hi))


SKIP_UNIFORM, SKIP_DECADE = 0, 1


def skip_edges(t: float, s: int, mode: int = SKIP_UNIFORM) -> np.ndarray:
    """fp32 band edges inside [0, t) for s successor models (P:541 / S:320)."""
    out = np.zeros(max(s - 1, 1), np.float32)
    lib().hso_skip_edges(float(t), int(s), int(mode), _ptr(out))
    return out[: max(s - 1, 0)]


def skip_band(c: float, edges: np.ndarray) -> int:
    e = np.ascontiguousarray(edges, dtype=np.float32)
    if e.size == 0:
        return 0
    return int(lib().hso_skip_band(float(c), _ptr(e), int(e.size + 1)))


def cascade_skip(conf_by_stage: np.ndarray, thresholds, mode: int = SKIP_UNIFORM):
    """(stage_of, visits bitmask) with skip connections."""
    c = np.ascontiguousarray(conf_by_stage, dtype=np.float64)
    K, n = c.shape
    t = np.zeros(K, np.float64)
    tt = np.asarray(thresholds, dtype=np.float64).reshape(-1)
    t[: min(K, tt.size)] = tt[: min(K, tt.size)]
    stage_of = np.empty(n, np.int32)
    visits = np.empty(n, np.uint32)
    lib().hso_cascade_skip(int(K), int(n), _ptr(c), _ptr(t), int(mode), _ptr(stage_of), _ptr(visits))
    return stage_of, visits


def skip_stage_lists(stage_of: np.ndarray, visits: np.ndarray, K: int):
    """Per model k: (batch = requests visiting k, accepted at k), increasing order."""
    return [(np.flatnonzero((visits >> k) & 1), np.flatnonzero(stage_of == k)) for k in range(K)]


def stage_lists(stage_of: np.ndarray, K: int):
    """Per-stage (batch, accepted, deferred) request lists, increasing order (D4)."""
    out = []
    for k in range(K):
        out.append((np.flatnonzero(stage_of >= k), np.flatnonzero(stage_of == k),
                    np.flatnonzero(stage_of > k)))
    return out


# --------------------------------------------------------------------------
# D5 calibration.  P:457-489 (Alg. 1, AP mode); exact sweep of SURVEY 8(c).
# --------------------------------------------------------------------------
def calibrate(conf: np.ndarray, correct: np.ndarray, log2_bins: int = 12, target: int = -1,
              refine_passes: int = 0):
    """conf[K-1, N] (fp64 or fp32), correct[K, N] (0/1) -> dict of b, t, reach, ..."""
    c = np.ascontiguousarray(conf, dtype=np.float64)
    ok = np.ascontiguousarray(correct, dtype=np.uint8)
    K = ok.shape[0]
    N = ok.shape[1]
    assert c.shape == (K - 1, N)
    b = np.empty(K - 1, np.int32)
    reach = np.empty(K, np.int64)
    handled = np.empty(K, np.int64)
    A = ctypes.c_int64()
    tau = ctypes.c_int64()
    rc = lib().hso_calibrate(int(K), int(N), _ptr(c), _ptr(ok), int(log2_bins), int(target),
                             int(refine_passes), _ptr(b), _ptr(reach), _ptr(handled),
                             ctypes.byref(A), ctypes.byref(tau))
    if rc != 0:
        raise ValueError("oracle: invalid calibration argument")
    B = 1 << log2_bins
    t = [float("inf") if int(x) == B + 1 else int(x) / B for x in b] + [0.0]
    return {"b": b, "t": np.array(t, np.float64), "reach": reach, "handled": handled,
            "correct_total": A.value, "tau": tau.value}


def bin_index(c, log2_bins: int):
    """bin(c) = min(B, floor(c * B)); NaN -> -1.  (D5 grid, reading G10.)"""
    B = 1 << log2_bins
    c = np.asarray(c, dtype=np.float64)
    out = np.floor(c * B)
    out = np.clip(out, 0, B)
    out = np.where(np.isnan(c), -1, out)
    return out.astype(np.int64)


# --------------------------------------------------------------------------
# NEXT-4: threshold performance graph, AP and EO (Alg. 1).
# --------------------------------------------------------------------------
def grid_size(K: int, log2_bins: int) -> int:
    """Threshold vectors on the D5 grid: (B+2)^(K-1)."""
    return ((1 << log2_bins) + 2) ** (K - 1)


def grid_vector(s: int, K: int, log2_bins: int) -> list:
    """Digits of grid vector s, b_0 most significant (itertools.product order)."""
    R = (1 << log2_bins) + 2
    b = []
    for _ in range(K - 1):
        b.append(s % R)
        s //= R
    return b[::-1]


def replay(conf: np.ndarray, correct: np.ndarray, log2_bins: int, weights, bvecs=None):
    """Alg. 1 line 4 for every threshold vector: (correct count, energy, reach[S, K]).
    conf[K-1, N], correct[K, N]; bvecs[S, K-1] grid indices or None = the whole grid."""
    c = np.ascontiguousarray(conf, dtype=np.float64)
    ok = np.ascontiguousarray(correct, dtype=np.uint8)
    K, N = ok.shape
    assert c.shape == (K - 1, N)
    if bvecs is None:
        S = grid_size(K, log2_bins)
        bv = None
    else:
        bv = np.ascontiguousarray(bvecs, dtype=np.int32).reshape(-1, K - 1)
        S = bv.shape[0]
    w = np.ascontiguousarray(weights, dtype=np.int64).reshape(K)
    oc = np.empty(S, np.int64)
    oe = np.empty(S, np.int64)
    orch = np.empty((S, K), np.int64)
    lib().hso_replay(int(K), int(N), _ptr(c), _ptr(ok), int(log2_bins), int(S),
                     None if bv is None else _ptr(bv), _ptr(w), _ptr(oc), _ptr(oe), _ptr(orch))
    return oc, oe, orch


def perf_graph(correct_s, energy_s, tau: int, floor: int):
    """The threshold performance graph's frontier and the AP / EO picks.

    Frontier (Alg. 1 output T, the curve of P:442-444): the Pareto set of the
    (correct count, energy) points -- for each correct count c the least energy
    of a vector with exactly c correct (lowest vector index on ties), kept iff
    strictly below the least energy of every larger count.  Ascending c.
    AP (G9): the least-energy vector with >= tau correct = the first
    frontier point with c >= tau.  EO (reading G23): among interior
    frontier points j with c_j >= floor (a >= a_{m_{n-1}}), the largest second
    divided difference of e(c),
        D_j = (e_{j+1} - e_j) / (c_{j+1} - c_j) - (e_j - e_{j-1}) / (c_j - c_{j-1})
    in fp64 (ties: lowest e); no interior candidate -> EO = AP.
    Returns dict(front_c, front_e, front_s, ap, eo) (ap / eo: vector index or -1)."""
    C = np.asarray(correct_s, dtype=np.int64)
    E = np.asarray(energy_s, dtype=np.int64)
    best = {}
    for s in range(C.size):
        c, e = int(C[s]), int(E[s])
        if c not in best or e < best[c][0]:
            best[c] = (e, s)
    front = []
    m = None
    for c in sorted(best, reverse=True):
        e, s = best[c]
        if m is None or e < m:
            front.append((c, e, s))
            m = e
    front.reverse()
    fc = np.array([f[0] for f in front], np.int64)
    fe = np.array([f[1] for f in front], np.int64)
    fs = np.array([f[2] for f in front], np.int64)
    ap = -1
    for j in range(len(front)):
        if fc[j] >= tau:
            ap = int(fs[j])
            break
    eo, best_d = -1, None
    for j in range(1, len(front) - 1):
        if fc[j] < floor:
            continue
        d = (float(fe[j + 1] - fe[j]) / float(fc[j + 1] - fc[j])
             - float(fe[j] - fe[j - 1]) / float(fc[j] - fc[j - 1]))
        if best_d is None or d > best_d:
            best_d, eo = d, int(fs[j])
    if eo < 0:
        eo = ap
    return {"front_c": fc, "front_e": fe, "front_s": fs, "ap": ap, "eo": eo}
