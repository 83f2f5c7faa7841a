"""Brute-force threshold calibration by cascade simulation -- TEST INFRASTRUCTURE ONLY.

A second, independent implementation of the D5 sweep that shares
no code with ``hs_oracle.c``: for every candidate threshold it replays the
whole cascade on the validation set (P:443-444 routing rule) and counts correct
answers, exactly as Alg. 1 line 4 "Compute a on D_v" evaluates a
threshold set.  O((B+2) * N * K) per move: tiny inputs only.
"""
from __future__ import annotations

import itertools
import math


def _bin(c: float, B: int) -> int:
    if c != c:  # NaN
        return -1
    return min(B, max(0, math.floor(c * B)))


def simulate(bins, correct, b):
    """Replay the cascade.  bins[k][r] (k < K-1), correct[k][r], b[k] threshold
    indices.  Returns (correct count, handled[k], reach[k])."""
    K = len(correct)
    N = len(correct[0])
    handled = [0] * K
    reach = [0] * K
    total = 0
    for r in range(N):
        k = 0
        reach[0] += 1
        while k < K - 1 and not (bins[k][r] >= b[k]):
            k += 1
            reach[k] += 1
        handled[k] += 1
        total += int(correct[k][r])
    return total, handled, reach


def greedy_by_simulation(conf, correct, log2_bins: int, target: int = -1):
    """Forward greedy: b_k = the smallest b whose cascade (b_1..b_{k-1}, b, defer
    all after k) keeps >= tau correct answers (AP)."""
    B = 1 << log2_bins
    K = len(correct)
    N = len(correct[0])
    bins = [[_bin(float(conf[k][r]), B) for r in range(N)] for k in range(K - 1)]
    tau = sum(int(x) for x in correct[K - 1]) if target < 0 else target
    b = [B + 1] * (K - 1)
    for k in range(K - 1):
        for cand in range(B + 2):
            trial = b[:k] + [cand] + [B + 1] * (K - 2 - k)
            if simulate(bins, correct, trial)[0] >= tau:
                b[k] = cand
                break
    total, handled, reach = simulate(bins, correct, b)
    return {"b": b, "correct_total": total, "handled": handled, "reach": reach, "tau": tau}


def refine_by_simulation(conf, correct, log2_bins: int, passes: int, target: int = -1):
    """D5's refinement by coordinate descent on the simulated cascade: starting
    from the greedy thresholds, each pass visits k = 1..K-1 in order and sets
    b_k = the smallest b whose cascade (b_k = b, every other threshold as it
    stands) still keeps >= tau correct answers -- Alg. 1's local search "Repeat
    line 3-4 on search space [k - eps, k + eps]" taken to its exact
    per-coordinate minimum.  Stops after ``passes`` passes or at a fixpoint."""
    B = 1 << log2_bins
    K = len(correct)
    N = len(correct[0])
    bins = [[_bin(float(conf[k][r]), B) for r in range(N)] for k in range(K - 1)]
    g = greedy_by_simulation(conf, correct, log2_bins, target)
    tau, b = g["tau"], list(g["b"])
    for _ in range(passes):
        changed = False
        for k in range(K - 1):
            for cand in range(B + 2):
                trial = b[:k] + [cand] + b[k + 1:]
                if simulate(bins, correct, trial)[0] >= tau:
                    if cand != b[k]:
                        b[k] = cand
                        changed = True
                    break
        if not changed:
            break
    total, handled, reach = simulate(bins, correct, b)
    return {"b": b, "correct_total": total, "handled": handled, "reach": reach, "tau": tau}


def exhaustive_min_energy(conf, correct, log2_bins: int, energy, target: int = -1):
    """Exhaustive grid search over all (B+2)^(K-1) threshold vectors: the AP
    point of minimal energy e = sum_k reach_k * e_k (reach reading of
    rho, G14); ties broken by the lexicographically smallest b."""
    B = 1 << log2_bins
    K = len(correct)
    N = len(correct[0])
    bins = [[_bin(float(conf[k][r]), B) for r in range(N)] for k in range(K - 1)]
    tau = sum(int(x) for x in correct[K - 1]) if target < 0 else target
    best = None
    for b in itertools.product(range(B + 2), repeat=K - 1):
        total, handled, reach = simulate(bins, correct, list(b))
        if total < tau:
            continue
        e = sum(reach[k] * energy[k] for k in range(K))
        if best is None or e < best[0]:
            best = (e, list(b), total)
    return {"energy": best[0], "b": best[1], "correct_total": best[2], "tau": tau}
