"""Synthetic cascade workloads (input generator shared by tests, smoke and bench).

``synth`` holds the numpy implementation and the workload families; this module
adds the GPU twin (``libhs_synth.so``) that writes the same bytes into torch
tensors for the large configurations.  No method arithmetic lives here.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .synth import FAMILIES, VAL_ID_BASE, Family, fam_logits_np, labels_np, logits_np, scaled  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libhs_synth.so")
_lock = threading.Lock()
_lib = None


def _synth_lib():
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(_LIB):
                raise ImportError(f"{_LIB} missing: run __graft_entry__.build()")
            L = ctypes.CDLL(_LIB)
            P, I64, I32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
            L.hs_synth_logits.argtypes = [P, I32, P, I64, I64, I32, I64, I64, I32, ctypes.c_uint32,
                                          I64, I32, P, P]
            L.hs_synth_logits.restype = I32
            L.hs_synth_labels.argtypes = [P, P, I64, I64, I32, I64, ctypes.c_uint32, P]
            L.hs_synth_labels.restype = I32
            _lib = L
    return _lib


def gpu_logits(out, fam: Family, stage: int, *, ids=None, id_base: int = 0, n: int | None = None,
               stream=None, scale_log2: int = 4):
    """Fill ``out`` ([n*L, stride] bf16/fp32 CUDA tensor) with stage ``stage`` logits
    for request ids ``ids`` (CUDA int64) or ``id_base + i``."""
    import torch
    n = int(n if n is not None else (ids.numel() if ids is not None else out.shape[0] // fam.L))
    dtype = 1 if out.dtype == torch.bfloat16 else 0
    s = (stream or torch.cuda.current_stream()).cuda_stream
    mg = (ctypes.c_int32 * 7)(*fam.margin)
    rc = _synth_lib().hs_synth_logits(out.data_ptr(), dtype, None if ids is None else ids.data_ptr(),
                                      int(id_base), n, fam.L, fam.C, out.stride(0), int(stage),
                                      fam.seed & 0xFFFFFFFF, fam.thr[stage], scale_log2, mg, s)
    if rc != 0:
        raise RuntimeError(f"hs_synth_logits failed: cuda error {rc}")
    return out


def gpu_labels(out, fam: Family, *, ids=None, id_base: int = 0, n: int | None = None, stream=None):
    import torch
    n = int(n if n is not None else out.numel() // fam.L)
    s = (stream or torch.cuda.current_stream()).cuda_stream
    rc = _synth_lib().hs_synth_labels(out.data_ptr(), None if ids is None else ids.data_ptr(),
                                      int(id_base), n, fam.L, fam.C, fam.seed & 0xFFFFFFFF, s)
    if rc != 0:
        raise RuntimeError(f"hs_synth_labels failed: cuda error {rc}")
    return out
