"""Pins for the oracle's routing (D3/D4) and calibration (D5).  CPU only.
Citations: P:443-444 (routing rule), P:457-489 (Alg. 1, AP)
(route_request / evaluate invariants), S:246/S:539 (grid search)."""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import bruteforce

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def test_hand_cascade():
    d = json.load(open(os.path.join(GOLD, "hand_cascade.json")))
    conf = np.array(d["conf"])
    K = d["K"]
    stage_of = oracle.cascade(conf, d["t"])
    assert list(stage_of) == d["stage_of"]
    lists = oracle.stage_lists(stage_of, K)
    for k in range(K):
        assert list(lists[k][1]) == d["accepted"][k]
        assert list(lists[k][2]) == d["deferred"][k]
    # the same lists by composing per-stage stable splits (what the GPU does)
    batch = np.arange(conf.shape[1])
    for k in range(K):
        acc, dfr = oracle.route(conf[k, batch], d["t"][k], k == K - 1)
        assert list(batch[acc]) == d["accepted"][k]
        assert list(batch[dfr]) == d["deferred"][k]
        batch = batch[dfr]


def test_fig3_narrative():
    """c = 0.2 < t = 0.7 is passed on; c = 0.7 stays (tie accepts, G5)."""
    acc, dfr = oracle.route(np.array([0.2, 0.7]), 0.7, False)
    assert list(acc) == [1] and list(dfr) == [0]


def test_route_invariants_random():
    rng = np.random.default_rng(0)
    for n in (0, 1, 17, 1000):
        c = rng.uniform(size=n)
        c[rng.uniform(size=n) < 0.05] = np.nan
        for t in (0.0, 0.3, 0.5, 1.0, np.inf):
            acc, dfr = oracle.route(c, t, False)
            assert len(acc) + len(dfr) == n
            assert len(np.intersect1d(acc, dfr)) == 0
            assert np.all(np.diff(acc) > 0) and np.all(np.diff(dfr) > 0)
            assert np.array_equal(acc, np.flatnonzero(c >= t))   # library special case
        # t = 0: everything answered by m_1 except invalid (NaN) rows (north_star)
        acc, dfr = oracle.route(c, 0.0, False)
        assert np.array_equal(dfr, np.flatnonzero(np.isnan(c)))
        # last stage accepts everything (G6)
        acc, dfr = oracle.route(c, 0.9, True)
        assert len(acc) == n and len(dfr) == 0


def test_cascade_invariants():
    """rho conservation, accuracy bounds, full escalation."""
    rng = np.random.default_rng(1)
    K, n = 4, 500
    conf = rng.uniform(size=(K, n))
    correct = (rng.uniform(size=(K, n)) < 0.7).astype(np.uint8)
    for t in ([0, 0, 0, 0], [np.inf] * 3 + [0], [0.5, 0.6, 0.7, 0]):
        s = oracle.cascade(conf, t)
        handled = np.bincount(s, minlength=K)
        assert handled.sum() == n
        acc = correct[s, np.arange(n)].sum()
        assert acc <= correct.max(axis=0).sum()
        if t[0] == 0:
            assert np.all(s == 0)
        if t[0] == np.inf:
            assert np.all(s == K - 1) and acc == correct[K - 1].sum()


def test_hand_calibration():
    d = json.load(open(os.path.join(GOLD, "hand_calibration.json")))
    conf = np.array(d["conf"])
    ok = np.array(d["correct"], np.uint8)
    q = d["log2_bins"]
    r = oracle.calibrate(conf, ok, q)
    assert r["tau"] == d["tau"]
    assert list(r["b"]) == d["b"]
    assert list(r["t"]) == d["t"]
    assert list(r["handled"]) == d["handled"] and list(r["reach"]) == d["reach"]
    B = 1 << q
    bins = [list(oracle.bin_index(conf[0], q))]
    got = [bruteforce.simulate(bins, ok, [b])[0] for b in range(B + 2)]
    assert got == d["cascade_correct_by_b"]


def _random_case(rng, K, N, correlated=True):
    d = rng.uniform(size=N)
    conf = np.empty((K - 1, N))
    ok = np.empty((K, N), np.uint8)
    for k in range(K):
        a = 0.5 + 0.1 * k
        ok[k] = (d + 0.3 * rng.normal(size=N) < a) if correlated else (rng.uniform(size=N) < a)
    for k in range(K - 1):
        conf[k] = np.clip(np.where(ok[k] == 1, rng.beta(5, 2, N), rng.beta(2, 3, N)), 0, 1)
        conf[k][rng.uniform(size=N) < 0.1] = rng.choice([0.0, 1.0, 0.5, 0.25])
    return conf, ok


def test_calibration_equals_simulation_bruteforce():
    """The sort-based sweep equals per-move cascade simulation (independent code)."""
    rng = np.random.default_rng(2024)
    for case in range(400):
        K = int(rng.integers(2, 5))
        N = int(rng.integers(1, 13))
        q = int(rng.integers(1, 4))
        conf, ok = _random_case(rng, K, N)
        if case % 7 == 0:
            conf[0, 0] = np.nan
        r = oracle.calibrate(conf, ok, q)
        bf = bruteforce.greedy_by_simulation(conf, ok, q)
        assert list(r["b"]) == bf["b"], (case, conf, ok)
        assert r["correct_total"] == bf["correct_total"]
        assert list(r["handled"]) == bf["handled"] and list(r["reach"]) == bf["reach"]
        assert r["correct_total"] >= r["tau"]            # AP guarantee


def test_k2_equals_exhaustive_optimum():
    """K=2: the sweep is the exact minimum-energy AP point on the grid (tightens S:539's 2%)."""
    rng = np.random.default_rng(77)
    for _ in range(200):
        N = int(rng.integers(1, 40))
        q = int(rng.integers(1, 5))
        conf, ok = _random_case(rng, 2, N)
        r = oracle.calibrate(conf, ok, q)
        ex = bruteforce.exhaustive_min_energy(conf, ok, q, energy=[1.0, 10.0])
        assert list(r["b"]) == ex["b"]


def test_refinement_never_raises_and_stays_feasible():
    rng = np.random.default_rng(5)
    for _ in range(200):
        K = int(rng.integers(3, 5))
        N = int(rng.integers(2, 30))
        q = int(rng.integers(1, 4))
        conf, ok = _random_case(rng, K, N)
        g = oracle.calibrate(conf, ok, q)
        r = oracle.calibrate(conf, ok, q, refine_passes=3)
        assert np.all(r["b"] <= g["b"])
        assert r["correct_total"] >= r["tau"]
        bins = [list(oracle.bin_index(conf[k], q)) for k in range(K - 1)]
        assert bruteforce.simulate(bins, ok, list(r["b"]))[0] == r["correct_total"]


def test_refinement_equals_simulation_coordinate_descent():
    """Pin for the oracle's refinement passes (D5, the analogue of Alg. 1's
    "Repeat line 3-4 on search space [k-eps, k+eps]"): bruteforce.py
    re-picks each b_k as the smallest b whose SIMULATED cascade keeps >= tau
    correct (independent code: no histograms, no suffix sums).  The cases are
    drawn so that refinement moves at least one threshold in many of them, so a
    refinement that does nothing (or moves the wrong coordinate) fails."""
    rng = np.random.default_rng(11)
    moved = 0
    for case in range(300):
        K = int(rng.integers(3, 6))
        N = int(rng.integers(2, 24))
        q = int(rng.integers(1, 4))
        conf, ok = _random_case(rng, K, N, correlated=True)
        if case % 9 == 0:
            conf[1, 0] = np.nan
        passes = int(rng.integers(1, 4))
        r = oracle.calibrate(conf, ok, q, refine_passes=passes)
        bf = bruteforce.refine_by_simulation(conf, ok, q, passes)
        assert list(r["b"]) == bf["b"], (case, passes, conf, ok)
        assert r["correct_total"] == bf["correct_total"] >= r["tau"]
        assert list(r["handled"]) == bf["handled"] and list(r["reach"]) == bf["reach"]
        moved += list(r["b"]) != list(oracle.calibrate(conf, ok, q)["b"])
    assert moved >= 20, moved


def test_refinement_hand_example():
    """Hand-worked K = 3, B = 2 (q = 1) case where refinement lowers b_1.
    c_1 = (.1, .9, .9) -> bins (0, 1, 1); c_2 = (.9, .9, .6) -> bins (1, 1, 1);
    correct m_1 = (0, 0, 0), m_2 = (1, 1, 0), m_3 = (0, 1, 0); tau = 1 (m_3).
    Greedy, k = 1 (later models defer all, so m_3 answers the rest): A = 0,
    G = 1, H = (0, -1, 0) over bins 0..2, S(0) = S(1) = -1, S(2) = 0, so
    b_1 = 2 (nobody is answered by m_1).  k = 2: G = 1, H[1] = 1, S(0) = 1 ->
    b_2 = 0 (m_2 answers all: 2 correct).  Refinement, k = 1, now that m_2
    answers whatever m_1 defers: b_1 = 0 answers everyone at m_1 (0 < tau);
    b_1 = 1 answers r1, r2 at m_1 and r0 at m_2 (1 >= tau): b_1 = 2 -> 1, and
    m_2's reach drops from 3 to 1."""
    conf = np.array([[0.1, 0.9, 0.9], [0.9, 0.9, 0.6]])
    ok = np.array([[0, 0, 0], [1, 1, 0], [0, 1, 0]], np.uint8)
    g = oracle.calibrate(conf, ok, 1)
    assert list(g["b"]) == [2, 0] and g["tau"] == 1 and g["correct_total"] == 2
    assert list(g["reach"]) == [3, 3, 0]
    r = oracle.calibrate(conf, ok, 1, refine_passes=1)
    assert list(r["b"]) == [1, 0] and r["correct_total"] == 1
    assert list(r["reach"]) == [3, 1, 0] and list(r["handled"]) == [2, 1, 0]


def test_explicit_target_and_defer_all():
    conf = np.array([[1.0, 1.0, 0.5]])
    ok = np.array([[0, 0, 1], [1, 1, 1]], np.uint8)
    r = oracle.calibrate(conf, ok, 3)
    # c = 1.0 is reachable; only b = B+1 (t = +inf, G11) defers the two wrong answers
    assert r["b"][0] == 9 and r["t"][0] == np.inf and r["correct_total"] == 3
    r = oracle.calibrate(conf, ok, 3, target=1)
    assert r["b"][0] == 0 and r["correct_total"] == 1


def test_bin_threshold_equivalence_fp32():
    """bin(c) >= b  <=>  c >= b/B exactly in fp32 (c*2^q is exact): calibrated
    thresholds route identically through the float test D3."""
    rng = np.random.default_rng(9)
    c = rng.uniform(size=200000).astype(np.float32)
    c[:1000] = np.float32(1.0)
    c[1000:2000] = (np.arange(1000) % 16 / 16).astype(np.float32)
    for q in (1, 4, 12, 14):
        B = 1 << q
        bins = oracle.bin_index(c, q)
        for b in rng.integers(0, B + 2, size=30):
            t = np.float32(b / B) if b <= B else np.float32(np.inf)
            assert np.array_equal(bins >= b, c >= t)


# ---------------------------------------------------------------------------
# NEXT-1 skip connections
# ---------------------------------------------------------------------------
def test_skip_golden():
    d = json.load(open(os.path.join(GOLD, "skip_bands.json")))
    np.testing.assert_allclose(oracle.skip_edges(0.7, 2, oracle.SKIP_UNIFORM), d["edges_uniform_t0.7_s2"], rtol=1e-7)
    np.testing.assert_allclose(oracle.skip_edges(0.7, 2, oracle.SKIP_DECADE), d["edges_decade_t0.7_s2"], rtol=1e-7)
    np.testing.assert_allclose(oracle.skip_edges(0.9, 4, oracle.SKIP_UNIFORM), d["edges_uniform_t0.9_s4"], rtol=1e-7)
    np.testing.assert_allclose(oracle.skip_edges(0.9, 4, oracle.SKIP_DECADE), d["edges_decade_t0.9_s4"], rtol=1e-6)
    K, t = d["K"], d["t"]
    for case in d["cases"]:
        mode = oracle.SKIP_UNIFORM if case["mode"] == "uniform" else oracle.SKIP_DECADE
        e = oracle.skip_edges(t[0], K - 1, mode)
        c1 = np.float32(case["c1"]).astype(np.float64)
        if "next" in case:
            assert 1 + oracle.skip_band(c1, e) == case["next"], case
        if "stage" in case:
            conf = np.array([[c1], [0.1], [0.9]])
            s, v = oracle.cascade_skip(conf, t, mode)
            assert s[0] == case["stage"]
            if "visits" in case:
                assert [k for k in range(K) if (v[0] >> k) & 1] == case["visits"]


def test_skip_reduces_to_sequential():
    """One successor (K=2) or all edges above every confidence -> plain cascade."""
    rng = np.random.default_rng(4)
    conf = rng.uniform(size=(2, 500))
    s1 = oracle.cascade(conf, [0.6, 0.0])
    s2, v = oracle.cascade_skip(conf, [0.6, 0.0])
    assert np.array_equal(s1, s2)


def test_skip_invariants_random():
    """Skips only jump forward; the answering model is >= the no-skip one's
    (S:206 'skip soundness'); visits are a subset of 0..stage; every request is
    answered exactly once (rho conservation)."""
    rng = np.random.default_rng(8)
    K, n = 5, 2000
    conf = rng.uniform(size=(K, n))
    conf[rng.uniform(size=(K, n)) < 0.01] = np.nan
    t = [0.6, 0.5, 0.7, 0.4, 0.0]
    seq = oracle.cascade(conf, t)
    for mode in (oracle.SKIP_UNIFORM, oracle.SKIP_DECADE):
        s, v = oracle.cascade_skip(conf, t, mode)
        assert np.all(s >= seq)
        assert np.all(v & 1)                                   # everyone starts at m_1
        assert np.all((v >> s) & 1) and np.all(v >> (s + 1) == 0)
        lists = oracle.skip_stage_lists(s, v, K)
        assert sum(len(a) for _, a in lists) == n
        # brute force: replay with explicit band lookups in Python
        for r in range(0, n, 37):
            k, path = 0, [0]
            while k < K - 1 and not (conf[k, r] >= t[k]):
                e = oracle.skip_edges(t[k], K - 1 - k, mode)
                k = k + 1 + int(sum(1 for x in e if not (conf[k, r] >= float(x))))
                path.append(k)
            assert k == s[r] and sum(1 << p for p in path) == v[r]
