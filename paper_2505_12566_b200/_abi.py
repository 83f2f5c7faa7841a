"""ctypes declarations of libhs.so (include/hs.h).  Argument marshalling only."""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
# HS_LIBHS selects an experiment build (A/B on one box); default is the product build
LIB_PATH = os.environ.get("HS_LIBHS") or os.path.join(_HERE, "libhs.so")

P = ctypes.c_void_p
I64 = ctypes.c_int64
I32 = ctypes.c_int32
F32 = ctypes.c_float
SZ = ctypes.c_size_t

HS_OK = 0
STATUS_NAMES = {0: "HS_OK", 1: "HS_ERR_INVALID_ARGUMENT", 2: "HS_ERR_NONFINITE_INPUT",
                3: "HS_ERR_CUDA", 4: "HS_ERR_NCCL", 5: "HS_ERR_WORKSPACE_TOO_SMALL", 6: "HS_ERR_UNSUPPORTED"}

# every symbol include/hs.h declares: name -> (restype, argtypes)
SIGNATURES = {
    "hs_confidence_workspace": (SZ, [I64, I32]),
    "hs_confidence": (I32, [P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, P, P, P, P, P, SZ, P, P]),
    "hs_confidence_topk": (I32, [P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, I32, P, P, P, P, P, SZ,
                                 P, P]),
    "hs_confidence_ex": (I32, [P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, I32, P, P, P, P, P, P,
                               SZ, P, P]),
    "hs_confidence_batched_workspace": (SZ, [I32, I64, I32]),
    "hs_confidence_batched": (I32, [P, P, I32, I32, I64, I32, I64, I64, P, I32, I32, P, P, P, P, P,
                                    SZ, P, P]),
    "hs_route_compact_workspace": (SZ, [I64]),
    "hs_route_compact": (I32, [P, I64, P, F32, P, I32, P, P, I32, P, P, P, P, P, P, I64, P, P, P,
                               SZ, P]),
    "hs_skip_edges": (I32, [F32, I32, I32, P]),
    "hs_skip_select": (I32, [P, I64, I32, P, P, P, SZ, P]),
    "hs_skip_route": (I32, [P, I64, P, F32, P, I32, I32, I32, P, P, I32, P, P, P, P, P, P, SZ, P]),
    "hs_cascade_step_workspace": (SZ, [I64, I32]),
    "hs_cascade_step": (I32, [I32, I32, P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, F32, P, P,
                              P, I64, P, P, P, P, P, P, P, SZ, P, P]),
    "hs_cascade_step_ex": (I32, [I32, I32, P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, F32, P, P,
                                 P, I64, P, P, P, P, P, P, P, SZ, P, I32, ctypes.c_uint32, P]),
    "hs_cascade_confidence": (I32, [I32, I32, P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, F32, P, P,
                                    P, SZ, P, I32, ctypes.c_uint32, P]),
    "hs_cascade_compact": (I32, [I32, I32, I64, I32, P, F32, P, P, P, I64, P, P, P, P, P, P, P, SZ, P]),
    "hs_calibrate_workspace": (SZ, [I32, I32]),
    "hs_calibrate_thresholds": (I32, [P, P, I32, I64, I32, I64, I32, P, P, P, P, P, P, SZ, P]),
    "hs_calibrate_begin": (I32, [I32, I32, I64, P, SZ, P]),
    "hs_calibrate_hist_ptr": (P, [P]),
    "hs_calibrate_hist_bytes": (SZ, [I32]),
    "hs_calibrate_histogram": (I32, [P, P, I32, I64, I32, I32, P, P, SZ, P]),
    "hs_calibrate_select": (I32, [I32, I32, I32, P, P, P, P, P, P, SZ, P]),
    "hs_fit_temperature_workspace": (SZ, [I32, I64]),
    "hs_fit_temperature": (I32, [P, I32, I32, I64, I64, I64, P, ctypes.c_double, ctypes.c_double, I32,
                                 P, P, P, P, P, SZ, P, P]),
    "hs_grid_size": (I64, [I32, I32]),
    "hs_grid_vector": (I32, [I64, I32, I32, P]),
    "hs_threshold_replay_workspace": (SZ, [I32, I64, I32]),
    "hs_threshold_replay": (I32, [P, P, I32, I64, I32, P, I64, P, P, P, P, P, P, SZ, P]),
    "hs_perf_graph_workspace": (SZ, [I64]),
    "hs_perf_graph": (I32, [P, P, I64, I64, I64, I64, P, I32, P, P, P, P, P, P, SZ, P, P]),
    "hs_peer_region_bytes": (SZ, [I32, I64, I64, I32]),
    "hs_peer_recv_ids": (P, [P, I32]),
    "hs_peer_recv_payload": (P, [P, I32]),
    "hs_peer_forward": (I32, [P, I32, P, P, P, P, I32, P, P, P]),
    "hs_peer_forward_publish": (I32, [P, P, P, P]),
    "hs_peer_forward_scatter": (I32, [P, I32, P, P, P, I32, P, P, P]),
    "hs_peer_forward_wait": (I32, [P, P, P]),
    "hs_calibrate_thresholds_peer": (I32, [P, P, I32, I64, I32, I64, P, P, P, P, P, P, P, SZ, P, P]),
    "hs_cascade_step_peer": (I32, [I32, I32, P, I32, I64, I32, I64, I64, P, P, F32, I32, I32, F32, P, P,
                                   P, I64, P, P, P, P, P, P, P, SZ, P, I32, ctypes.c_uint32, P, I32, P,
                                   I32, P, P]),
    "hs_ipc_alloc": (I32, [SZ, P]),
    "hs_ipc_free": (I32, [P]),
    "hs_ipc_handle": (I32, [P, P]),
    "hs_ipc_open": (I32, [P, P]),
    "hs_ipc_close": (I32, [P]),
    "hs_comm_unique_id": (I32, [P]),
    "hs_comm_create": (I32, [P, I32, I32, I32, P]),
    "hs_comm_destroy": (I32, [P]),
    "hs_calibrate_thresholds_comm": (I32, [P, P, I32, I64, I32, I64, P, P, P, P, P, P, P, SZ, P]),
    "hs_calibrate_thresholds_comm_ex": (I32, [P, P, I32, I64, I32, I64, I32, P, P, P, P, P, P, P, SZ, P]),
    "hs_forward_nccl_workspace": (SZ, [I32]),
    "hs_forward_nccl": (I32, [P, P, I64, P, P, I32, P, P, I64, P, P, P, SZ, P]),
    "hs_status_string": (ctypes.c_char_p, [I32]),
    "hs_last_error": (ctypes.c_char_p, []),
    "hs_launch_count": (ctypes.c_uint64, []),
    "hs_build_info": (ctypes.c_char_p, []),
}

PEER_MAX_WORLD = 8


class PeerGroup(ctypes.Structure):
    """hs_peer_t (include/hs.h): the peer-memory group as seen by this process."""
    _fields_ = [("rank", ctypes.c_int32), ("world", ctypes.c_int32), ("cap", ctypes.c_int64),
                ("payload_row_bytes", ctypes.c_int64), ("log2_bins", ctypes.c_int32),
                ("region", ctypes.c_void_p * PEER_MAX_WORLD)]


_lock = threading.Lock()
_lib = None


class HsError(RuntimeError):
    def __init__(self, fn: str, code: int, detail: str):
        super().__init__(f"{fn}: {STATUS_NAMES.get(code, code)}: {detail}")
        self.code = code


def lib():
    """Load libhs.so (built in-tree by __graft_entry__.build()).  There is no
    fallback: the router runs on the CUDA kernels or not at all."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ImportError(f"{LIB_PATH} is missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
            L = ctypes.CDLL(LIB_PATH)
            for name, (res, args) in SIGNATURES.items():
                f = getattr(L, name)
                f.restype = res
                f.argtypes = args
            if b"EXPERIMENT" in L.hs_build_info() and os.environ.get("HS_ALLOW_EXPERIMENT") != "1":
                raise ImportError(f"{LIB_PATH} is a timing-bound experiment build (wrong results); "
                                  "set HS_ALLOW_EXPERIMENT=1 to load it for A/B timing")
            _lib = L
    return _lib


def check(fn: str, code: int):
    if code != HS_OK:
        raise HsError(fn, code, lib().hs_last_error().decode(errors="replace"))


def call(fn: str, *args):
    check(fn, getattr(lib(), fn)(*args))
