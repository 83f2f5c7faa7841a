"""Seeded synthetic cascade workloads -- shared INPUT GENERATOR.

This module holds none of the method's arithmetic (no softmax, no confidence,
no routing, no calibration): it only fabricates the bytes a cascade of models
m_1..m_K would hand the router (per-stage logits keyed by request id) and the
validation labels.  Both the CUDA path's tests/bench and the oracle consume it;
it is the one module they share.  The same counter-based integer generator is
implemented twice, bit-identically: here in numpy (CPU) and in
``workload/csrc/synth.cu`` (GPU, used for the large configs).

Recipe (SURVEY 8(d) adapted to integer arithmetic so
both implementations agree bit for bit):

* keys: ``mix32`` (a 32-bit avalanche hash) of (seed, stage, request id, token,
  class).  Output is identical for any batch composition, order or GPU count.
* background logit of class j: code = (sum of the 4 bytes of h_j - 510) >> 3,
  an Irwin-Hall approximation of N(0, 18.5^2) in [-64, 63].
* request-level: label y ~ U[0, C) per token, latent difficulty d ~ U[0, 2^16)
  shared by all stages; stage noise e_k ~ U[0, 2^15).  The model is
  "meant" to be right iff d + e_k < thr_k, thr_k set from the family's
  marginal accuracy a_k (Table II).  Overlap across stages is
  therefore "not strictly subset".
* the winning class (y if meant right, else a random other class) gets code
  rb + U[0,rm1] + U[0,rm2] (+ min(slack >> cs, ccap) when cs > 0, slack =
  thr_k - d - e_k: requests far from the model's accuracy boundary are answered
  more confidently) when right, wb + U[0,wm] when wrong: confident answers are
  more often right.  Legacy profile (60,127,63,60,63,0,0); ViT families
  use VIT_MARGIN, tuned toward Table III's handled fractions.  Token models (L > 1): a wrong sequence has one
  wrong, low-margin token.
* value = code * 2^-scale_log2, exactly representable in bf16 and fp32.
  Whether the model is actually right is decided by the router's own argmax.
"""
from __future__ import annotations

import dataclasses
import math

import numpy as np

M32 = np.uint64(0xFFFFFFFF)
VAL_ID_BASE = 1 << 32          # validation request ids live above 2^32


def mix32(x):
    """lowbias32 avalanche hash on uint32 (numpy arrays or scalars)."""
    x = np.asarray(x, dtype=np.uint32)
    with np.errstate(over="ignore"):
        x = x ^ (x >> np.uint32(16))
        x = x * np.uint32(0x7FEB352D)
        x = x ^ (x >> np.uint32(15))
        x = x * np.uint32(0x846CA68B)
        x = x ^ (x >> np.uint32(16))
    return x


def _u32(v):
    return np.uint32(int(v) & 0xFFFFFFFF)


def seed_key(seed: int):
    return mix32(_u32(seed) ^ np.uint32(0x5BD1E995))


def stage_key(seed: int, stage: int):
    return mix32(seed_key(seed) ^ mix32(_u32(stage + 0x27D4EB2F)))


def _id_key(base, ids):
    ids = np.asarray(ids, dtype=np.int64).astype(np.uint64)
    lo = (ids & M32).astype(np.uint32)
    hi = (ids >> np.uint64(32)).astype(np.uint32)
    return mix32(mix32(base ^ lo) ^ hi)


def req_key(seed: int, ids):
    return _id_key(seed_key(seed), ids)


def row_key(seed: int, stage: int, ids):
    return _id_key(stage_key(seed, stage), ids)


def tok_key(rk, t):
    with np.errstate(over="ignore"):
        return mix32(rk + np.uint32(t) * np.uint32(0x9E3779B9))


def accuracy_threshold(a: float) -> int:
    """thr with P(d + e < thr) = a for d ~ U{0..65535}, e ~ U{0..32767} (continuous approx)."""
    A, Bw = 65536.0, 32768.0
    a = min(max(a, 0.0), 1.0)
    lo_area = Bw / (2 * A)                 # mass below x = Bw
    if a <= lo_area:
        x = math.sqrt(2 * a * A * Bw)
    elif a <= 1 - lo_area:
        x = Bw / 2 + a * A
    else:
        x = A + Bw - math.sqrt(2 * (1 - a) * A * Bw)
    return int(round(x))


def labels_np(seed: int, ids, L: int, C: int) -> np.ndarray:
    """int32 labels[n, L]."""
    rq = req_key(seed, ids)[:, None]
    t = np.arange(L, dtype=np.uint32)[None, :]
    return (mix32(rq ^ mix32(t + np.uint32(0x01000193))) % np.uint32(C)).astype(np.int32)


LEGACY_MARGIN = (60, 127, 63, 60, 63, 0, 0)


def winner_code(ok, slack, m1, m2, margin):
    """Code of the winning class (numpy, int64 arrays).  margin = (rb, rm1, rm2,
    wb, wm, cs, ccap): a right token gets rb + (m1 & rm1) + (m2 & rm2) plus, when
    cs > 0, min(max(slack, 0) >> cs, ccap) -- the further the request is from
    the model's accuracy boundary (slack = thr - d - e), the more confident the
    right answer; a wrong token gets wb + (m1 & wm).  Codes stay <= 255 so the
    values are exact in bf16."""
    rb, rm1, rm2, wb, wm, cs, ccap = margin
    right = rb + (m1 & rm1) + (m2 & rm2)
    if cs > 0:
        right = right + np.minimum(np.maximum(slack, 0) >> cs, ccap)
    return np.where(ok, right, wb + (m1 & wm))


def logits_np(seed: int, stage: int, ids, L: int, C: int, thr: int, dtype: str = "bf16",
              scale_log2: int = 4, margin=LEGACY_MARGIN) -> np.ndarray:
    """Stage ``stage`` logits for requests ``ids``: float32 [n*L, C], or raw bf16
    bits (uint16) [n*L, C] when dtype == 'bf16'."""
    ids = np.asarray(ids, dtype=np.int64)
    n = ids.size
    rq = req_key(seed, ids)
    rk = row_key(seed, stage, ids)
    d = mix32(rq ^ np.uint32(0xD1FF)) & np.uint32(0xFFFF)
    e = mix32(rk ^ np.uint32(0xE751)) & np.uint32(0x7FFF)
    meant = (d.astype(np.int64) + e.astype(np.int64)) < thr                   # [n]
    tstar = (mix32(rk ^ np.uint32(0x7777)) % np.uint32(L)).astype(np.int64)   # [n]
    lab = labels_np(seed, ids, L, C)                                          # [n, L]
    t = np.arange(L, dtype=np.uint32)[None, :]
    tk = tok_key(rk[:, None], t)                                              # [n, L]
    tok_ok = meant[:, None] | (np.arange(L)[None, :] != tstar[:, None])
    other = (mix32(tk ^ np.uint32(0x0BAD)) % np.uint32(max(C - 1, 1))).astype(np.int64)
    winner = np.where(tok_ok, lab, (lab.astype(np.int64) + 1 + other) % C).astype(np.int64)
    m1 = (mix32(tk ^ np.uint32(0x11))).astype(np.int64)
    m2 = (mix32(tk ^ np.uint32(0x22))).astype(np.int64)
    slack = (thr - d.astype(np.int64) - e.astype(np.int64))[:, None]
    wcode = winner_code(tok_ok, slack, m1, m2, margin)
    j = np.arange(C, dtype=np.uint32)[None, None, :]
    with np.errstate(over="ignore"):
        h = mix32(tk[:, :, None] + (j + np.uint32(1)) * np.uint32(0x85EBCA6B))
    s = ((h & np.uint32(255)) + ((h >> np.uint32(8)) & np.uint32(255)) +
         ((h >> np.uint32(16)) & np.uint32(255)) + (h >> np.uint32(24))).astype(np.int32)
    code = (s - 510) >> 3
    nl = n * L
    code = code.reshape(nl, C)
    code[np.arange(nl), winner.reshape(nl)] = wcode.reshape(nl)
    vals = code.astype(np.float32) * np.float32(2.0 ** -scale_log2)
    if dtype == "fp32":
        return vals
    return (vals.view(np.uint32) >> np.uint32(16)).astype(np.uint16)   # exact: <= 8 significant bits


def bf16_bits_to_f32(bits: np.ndarray) -> np.ndarray:
    return (bits.astype(np.uint32) << np.uint32(16)).view(np.float32)


# ViT families: the right answer's margin grows with the request's distance
# from the model's accuracy boundary, so confident-but-wrong and unsure-but-
# right answers overlap and AP calibration has to defer about half of the
# requests (tools/tune_generator.py).  C2 at full size: calibrated reach
# [1, .481, .312, .232, .182] (sum 2.21); handled 51.9 / 16.9 / 8.0 / 5.0 /
# 18.2 % -- Table III's ViT split is 59.6 / 5.1 / 18.2 / 17.1 %.
VIT_MARGIN = (50, 15, 7, 60, 63, 8, 180)

# --------------------------------------------------------------------------
# Workload families (BASELINE.json configs).
# --------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Family:
    name: str
    n: int                      # requests (or sequences) routed
    C: int                      # classes / vocabulary
    L: int                      # tokens per sequence (1 = classification / next token)
    dtype: str                  # "bf16" | "fp32"
    acc: tuple                  # marginal accuracies a_1..a_K (Table II)
    temps: tuple                # per-stage temperature T_k
    kind: int                   # 0 MAXPROB, 1 MAXPROB_SQ, 2 ENTROPY
    reduce: int                 # 0 NONE, 1 MIN, 2 MEAN
    n_val: int                  # validation samples for calibration
    payload_bytes: int = 0      # deferred-request payload row (bytes)
    log2_bins: int = 12
    seed: int = 0x250512566
    top_k: int = 0              # NEXT-2: stage confidence over the top_k logits (0 = full)
    margin: tuple = LEGACY_MARGIN   # winner-code profile (winner_code); ViT families: VIT_MARGIN

    @property
    def K(self):
        return len(self.acc)

    @property
    def thr(self):
        return tuple(accuracy_threshold(a) for a in self.acc)

    @property
    def elt_bytes(self):
        return 2 if self.dtype == "bf16" else 4

    @property
    def row_bytes(self):
        return self.L * self.C * self.elt_bytes


FAMILIES = {
    # C1: 2-stage ViT-S -> ViT-L, fp32, 4,096 x 1,000
    "c1": Family("c1_vit2_fp32", 4096, 1000, 1, "fp32", (0.808, 0.823), (1.0, 1.0), 0, 0, 4096,
                 seed=0x250512566 + 1, margin=VIT_MARGIN),
    # C2: 5-stage ViT family, bf16, 262,144 x 1,000, 50,000 validation
    "c2": Family("c2_vit5_bf16", 262144, 1000, 1, "bf16", (0.748, 0.808, 0.812, 0.813, 0.823),
                 (1.0, 1.1, 0.9, 1.0, 1.2), 0, 0, 50000, seed=0x250512566 + 2,
                 margin=VIT_MARGIN),
    # C3: 4-size T5, 16,384 seq x 64 tok x 32,128 vocab bf16, MIN over tokens
    "c3": Family("c3_t5x4_bf16", 16384, 32128, 64, "bf16", (0.782, 0.842, 0.871, 0.905),
                 (1.0, 1.0, 1.0, 1.0), 0, 1, 4096, payload_bytes=256, seed=0x250512566 + 3),
    # C4: Llama-like next token, 8,192 x 128,256 bf16, entropy confidence, 8 KB hidden payload
    "c4": Family("c4_llama3_bf16", 8192, 128256, 1, "bf16", (0.311, 0.369, 0.423),
                 (1.0, 1.0, 1.0), 2, 0, 8192, payload_bytes=8192, seed=0x250512566 + 4),
    # C5: streaming 5-stage ViT, 2^23 requests x 1,000 bf16 (sharded over GPUs)
    "c5": Family("c5_vit5_stream_bf16", 1 << 23, 1000, 1, "bf16",
                 (0.748, 0.808, 0.812, 0.813, 0.823), (1.0, 1.1, 0.9, 1.0, 1.2), 0, 0, 1 << 20,
                 seed=0x250512566 + 5, margin=VIT_MARGIN),
}


def fam_logits_np(f: Family, stage: int, ids, dtype: str | None = None, L: int | None = None,
                  C: int | None = None) -> np.ndarray:
    """logits_np with the family's seed, accuracy threshold and margin profile."""
    return logits_np(f.seed, stage, ids, L or f.L, C or f.C, f.thr[stage], dtype or f.dtype,
                     margin=f.margin)


def scaled(f: Family, n: int | None = None, n_val: int | None = None, C: int | None = None,
           L: int | None = None) -> Family:
    """A smaller copy of a family (parity tests at sizes the oracle finishes quickly)."""
    return dataclasses.replace(f, n=n or f.n, n_val=n_val or f.n_val, C=C or f.C, L=L or f.L)
