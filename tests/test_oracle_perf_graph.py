"""Pins for the oracle's threshold performance graph (NEXT-4; Alg. 1):
replay of threshold vectors, the Pareto frontier, AP and EO picks.  CPU only.

Independent references: the hand-worked graph (tests/golden/hand_perf_graph.json),
the pure-Python cascade simulation of oracle/bruteforce.py (shares no code with
hs_oracle.c), the closed forms of the all-accept / defer-all vectors, D5's
calibration (K = 2 exact optimum), and closed-form EO curves."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import bruteforce

GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


def test_hand_graph():
    d = json.load(open(os.path.join(GOLD, "hand_perf_graph.json")))
    conf = np.array(d["conf"], np.float32)
    ok = np.array(d["correct"], np.uint8)
    c, e, reach = oracle.replay(conf, ok, d["log2_bins"], d["weights"])
    assert c.tolist() == d["correct_by_b"]
    assert e.tolist() == d["energy_by_b"]
    assert reach.tolist() == d["reach_by_b"]
    g = oracle.perf_graph(c, e, d["tau"], floor=int(ok[0].sum()))
    assert g["front_c"].tolist() == d["front_c"] and g["front_e"].tolist() == d["front_e"]
    assert g["front_s"].tolist() == d["front_s"]
    assert g["ap"] == d["ap"] and g["eo"] == d["eo"]
    cal = oracle.calibrate(conf, ok, d["log2_bins"])
    assert oracle.grid_vector(g["ap"], 2, d["log2_bins"]) == cal["b"].tolist()


def _case(rng, K, N, q, nan=False):
    conf = rng.random((K - 1, N)).astype(np.float32)
    conf[rng.random((K - 1, N)) < 0.15] = np.float32(1.0)
    if nan:
        conf[0, 0] = np.nan
    # correctness correlated with confidence (the cascade's premise)
    ok = np.zeros((K, N), np.uint8)
    for k in range(K):
        base = conf[min(k, K - 2)] if k < K - 1 else rng.random(N)
        ok[k] = (rng.random(N) < 0.3 + 0.6 * np.nan_to_num(base)).astype(np.uint8)
    w = rng.integers(1, 50, size=K).astype(np.int64)
    w.sort()
    return conf, ok, w


def test_replay_equals_bruteforce_simulation():
    rng = np.random.default_rng(11)
    for trial in range(120):
        K = int(rng.integers(2, 5))
        N = int(rng.integers(1, 13))
        q = int(rng.integers(1, 3))
        conf, ok, w = _case(rng, K, N, q, nan=trial % 7 == 0)
        c, e, reach = oracle.replay(conf, ok, q, w)
        B = 1 << q
        bins = [[bruteforce._bin(float(conf[k][r]), B) for r in range(N)] for k in range(K - 1)]
        for s in range(oracle.grid_size(K, q)):
            b = oracle.grid_vector(s, K, q)
            tot, handled, rch = bruteforce.simulate(bins, ok, b)
            assert c[s] == tot and reach[s].tolist() == rch
            assert e[s] == sum(rch[k] * int(w[k]) for k in range(K))


def test_grid_order_is_itertools_product():
    import itertools
    got = [oracle.grid_vector(s, 4, 1) for s in range(oracle.grid_size(4, 1))]
    assert got == [list(b) for b in itertools.product(range(4), repeat=3)]


def test_all_accept_and_defer_all_closed_forms():
    rng = np.random.default_rng(12)
    conf, ok, w = _case(rng, 4, 500, 3, nan=True)
    N = 500
    B = 8
    bv = np.array([[0, 0, 0], [B + 1, B + 1, B + 1]], np.int32)
    c, e, reach = oracle.replay(conf, ok, 3, w, bvecs=bv)
    nan0 = np.isnan(conf[0])
    # t = 0 at stage 1: every request with a finite confidence is answered by m_1
    # (north_star); the one NaN confidence (request 0) is deferred and m_2 answers it
    assert nan0.tolist() == [True] + [False] * (N - 1)
    assert reach[0].tolist() == [N, 1, 0, 0]
    assert c[0] == int(ok[0][1:].sum()) + int(ok[1][0])
    assert e[0] == N * int(w[0]) + int(w[1])
    # defer all: everything reaches and is answered by m_K
    assert reach[1].tolist() == [N] * 4 and c[1] == int(ok[3].sum()) and e[1] == N * int(w.sum())


def test_exhaustive_ap_equals_bruteforce_min_energy():
    rng = np.random.default_rng(13)
    for _ in range(60):
        K = int(rng.integers(2, 5))
        N = int(rng.integers(2, 12))
        q = int(rng.integers(1, 3))
        conf, ok, w = _case(rng, K, N, q)
        c, e, _ = oracle.replay(conf, ok, q, w)
        tau = int(ok[K - 1].sum())
        g = oracle.perf_graph(c, e, tau, floor=int(ok[K - 2].sum()))
        bf = bruteforce.exhaustive_min_energy(conf, ok, q, [int(x) for x in w])
        assert e[g["ap"]] == bf["energy"]
        assert oracle.grid_vector(g["ap"], K, q) == bf["b"]


def test_k2_exhaustive_ap_is_the_calibration():
    """D5: for K = 2 the forward sweep is the exact grid optimum (w_1 < w_2)."""
    rng = np.random.default_rng(14)
    for _ in range(40):
        conf, ok, w = _case(rng, 2, int(rng.integers(5, 300)), 3)
        c, e, _ = oracle.replay(conf, ok, 3, w)
        g = oracle.perf_graph(c, e, int(ok[1].sum()), floor=int(ok[0].sum()))
        cal = oracle.calibrate(conf, ok, 3)
        assert oracle.grid_vector(g["ap"], 2, 3) == cal["b"].tolist()
        assert c[g["ap"]] == cal["correct_total"]


def test_greedy_never_beats_the_exhaustive_optimum():
    rng = np.random.default_rng(15)
    for _ in range(30):
        conf, ok, w = _case(rng, 4, int(rng.integers(20, 200)), 2)
        c, e, _ = oracle.replay(conf, ok, 2, w)
        g = oracle.perf_graph(c, e, int(ok[3].sum()), floor=int(ok[2].sum()))
        cal = oracle.calibrate(conf, ok, 2)
        cg, eg, _ = oracle.replay(conf, ok, 2, w, bvecs=cal["b"][None, :])
        assert cg[0] >= int(ok[3].sum())
        assert e[g["ap"]] <= eg[0] and c[g["ap"]] >= int(ok[3].sum())


def test_frontier_is_the_pareto_set():
    rng = np.random.default_rng(16)
    conf, ok, w = _case(rng, 3, 150, 3)
    c, e, _ = oracle.replay(conf, ok, 3, w)
    g = oracle.perf_graph(c, e, 0, 0)
    fc, fe, fs = g["front_c"], g["front_e"], g["front_s"]
    assert (np.diff(fc) > 0).all() and (np.diff(fe) > 0).all()
    assert (c[fs] == fc).all() and (e[fs] == fe).all()
    for s in range(c.size):      # every point is weakly dominated by a frontier point
        assert ((fc >= c[s]) & (fe <= e[s])).any()
    for j in range(fc.size):     # and no point strictly dominates a frontier point
        dom = (c >= fc[j]) & (e <= fe[j]) & ((c > fc[j]) | (e < fe[j]))
        assert not dom.any()
        # representative = the lowest index with that (c, e)
        assert fs[j] == np.flatnonzero((c == fc[j]) & (e == fe[j]))[0]


def test_eo_closed_forms():
    cs = np.arange(21, dtype=np.int64)
    kink = np.where(cs <= 10, cs, 10 + 5 * (cs - 10)).astype(np.int64)
    g = oracle.perf_graph(cs, kink, tau=20, floor=0)
    assert g["eo"] == 10 and g["ap"] == 20          # the knee of e(a); AP at full accuracy
    g = oracle.perf_graph(cs, kink, tau=20, floor=11)
    assert g["eo"] == 11                            # all D_j = 0 above the floor: lowest e
    quad = cs * cs                                  # constant second difference: lowest e
    assert oracle.perf_graph(cs, quad, tau=20, floor=0)["eo"] == 1
    assert oracle.perf_graph(cs, quad, tau=20, floor=7)["eo"] == 7
    # dominated points do not enter the frontier; EO is a frontier vector
    c2 = np.concatenate([cs, cs])
    e2 = np.concatenate([kink + 3, kink])
    g = oracle.perf_graph(c2, e2, tau=20, floor=0)
    assert g["eo"] == 21 + 10 and g["ap"] == 21 + 20
    # fewer than three frontier points: EO = AP
    g = oracle.perf_graph(np.array([2, 3]), np.array([4, 14]), tau=3, floor=0)
    assert g["eo"] == g["ap"] == 1
