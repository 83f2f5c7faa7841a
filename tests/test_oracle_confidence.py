"""Pins for the oracle's confidence (D1/D2): closed forms, library special cases,
invariants.  CPU only.  Citations: P:373-391 (TS, Eq. 1), P:413-430 (per-task
confidence), S:124-150 (SPEC examples and invariants)."""
import json
import math
import os

import numpy as np
import pytest
import scipy.special
import torch

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _bf16_bits(x: np.ndarray) -> np.ndarray:
    return torch.from_numpy(np.asarray(x, np.float32)).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)


def test_golden_closed_forms():
    d = json.load(open(os.path.join(GOLD, "conf_closed_forms.json")))
    for case in d["cases"]:
        p, H, am = oracle.row_stats(case["logits"], case["T"])
        assert am == case["argmax"]
        assert p == pytest.approx(case["p_max"], rel=1e-14, abs=0)
        assert p * p == pytest.approx(case["p_max_sq"], rel=1e-14, abs=0)
        assert math.exp(-H) == pytest.approx(case["exp_neg_H"], rel=1e-13, abs=1e-300)


@pytest.mark.parametrize("k", [2, 3, 4, 7, 1000, 32128])
@pytest.mark.parametrize("T", [0.05, 1.0, 20.0])
def test_uniform_over_k(k, T):
    """uniform over k -> p_max = exp(-H) = 1/k, H = ln k (S:125 symmetry)."""
    p, H, am = oracle.row_stats(np.full(k, 1.25), T)
    assert p == pytest.approx(1.0 / k, rel=1e-13)
    assert H == pytest.approx(math.log(k), rel=1e-12)
    assert am == 0


def test_uniform_support_with_masked_classes():
    """-inf entries are masked classes: uniform over the k finite ones (G-readings, S:122 ext.)."""
    x = np.full(10, -np.inf)
    x[[2, 5, 7]] = 0.3
    p, H, am = oracle.row_stats(x, 1.0)
    assert p == pytest.approx(1 / 3, rel=1e-14)
    assert H == pytest.approx(math.log(3), rel=1e-13)
    assert am == 2


@pytest.mark.parametrize("d,T", [(0.0, 1.0), (1.0, 1.0), (4.0, 2.5), (30.0, 0.7), (1e-3, 3.0)])
def test_two_classes_sigmoid(d, T):
    """C=2 -> p_max = sigmoid(|x1-x0|/T); H = binary entropy."""
    p, H, am = oracle.row_stats([0.1, 0.1 + d], T)
    s = 1.0 / (1.0 + math.exp(-d / T))
    assert p == pytest.approx(s, rel=1e-14)
    q = 1 - s
    Hb = -(s * math.log(s) + (q * math.log(q) if q > 0 else 0.0))
    assert H == pytest.approx(Hb, rel=1e-9, abs=1e-15)
    assert am == (1 if d > 0 else 0)


def test_saturated_is_exactly_one():
    """(1000,0,0) -> exactly 1.0 in fp64 -- why 'defer all' needs index B+1 (G11)."""
    p, H, am = oracle.row_stats([1000.0, 0.0, 0.0], 1.0)
    assert p == 1.0 and am == 0 and H >= 0


def test_library_special_cases_random_rows():
    """fp64 torch.softmax / scipy logsumexp / Categorical.entropy on random rows."""
    rng = np.random.default_rng(1234)
    for C in (2, 5, 1000, 4099):
        for T in (0.05, 0.5, 1.0, 7.0):
            x = rng.normal(0, 3, size=C)
            p, H, am = oracle.row_stats(x, T)
            t = torch.from_numpy(x / T)
            sm = torch.softmax(t, dim=0)
            assert p == pytest.approx(float(sm.max()), rel=1e-12)
            assert am == int(torch.argmax(t))
            assert -math.log(p) == pytest.approx(scipy.special.logsumexp(x / T) - x.max() / T, rel=1e-10, abs=1e-13)
            ent = float(torch.distributions.Categorical(logits=t).entropy())
            assert H == pytest.approx(ent, rel=1e-9, abs=1e-12)


def test_scale_invariance():
    """c(alpha x, alpha T) = c(x, T)  (temperature absorbs global scale)."""
    rng = np.random.default_rng(7)
    for _ in range(50):
        x = rng.normal(0, 2, size=37)
        a = float(rng.uniform(0.1, 10))
        T = float(rng.uniform(0.2, 5))
        p1, H1, a1 = oracle.row_stats(x, T)
        p2, H2, a2 = oracle.row_stats(a * x, a * T)
        assert a1 == a2
        assert p1 == pytest.approx(p2, rel=1e-12)
        assert H1 == pytest.approx(H2, rel=1e-10, abs=1e-14)


def test_argmax_invariance_and_range():
    """S:147 / acceptance 1: argmax unchanged by temperature; S:148 range [0,1]."""
    rng = np.random.default_rng(99)
    n, C = 2000, 16
    x = rng.normal(0, 2, size=(n, C)).astype(np.float32)
    ref = oracle.confidence(x, n, 1, C, C, 1.0)["argmax"]
    assert np.array_equal(ref, np.argmax(x, axis=1))
    for T in np.geomspace(0.02, 50, 25):
        for kind in (oracle.MAXPROB, oracle.MAXPROB_SQ, oracle.ENTROPY):
            r = oracle.confidence(x, n, 1, C, C, float(T), kind=kind)
            assert np.array_equal(r["argmax"], ref)
            assert np.all(r["conf"] >= 1.0 / C - 1e-15) if kind != oracle.MAXPROB_SQ else True
            assert np.all((r["conf"] >= 0) & (r["conf"] <= 1.0))


def test_ties_lowest_index():
    """G12: argmax ties -> lowest index (numpy/torch first occurrence)."""
    x = np.array([1.0, 3.0, 2.0, 3.0, 3.0])
    assert oracle.row_stats(x, 1.0)[2] == 1


@pytest.mark.parametrize("bad", [[np.nan, 0.0, 1.0], [0.0, np.inf, 1.0], [-np.inf, -np.inf]])
def test_invalid_rows(bad):
    """S:122 requires finite logits: NaN / +inf / all -inf rows are flagged."""
    assert oracle.row_stats(bad, 1.0) is None
    r = oracle.confidence(np.array(bad, np.float32), 1, 1, len(bad), len(bad), 1.0)
    assert r["bad"][0] == 1 and math.isnan(r["conf"][0])


def test_argument_errors():
    with pytest.raises(ValueError):
        oracle.confidence(np.zeros(4, np.float32), 4, 1, 1, 1, 1.0)      # C < 2
    with pytest.raises(ValueError):
        oracle.confidence(np.zeros(4, np.float32), 2, 1, 2, 2, 0.0)      # T <= 0
    with pytest.raises(ValueError):
        oracle.confidence(np.zeros(8, np.float32), 2, 2, 2, 2, 1.0)      # NONE with L > 1


def test_bf16_bits_equal_float_values():
    """bf16 input path widens exactly: same result as the fp32 copy of the values."""
    rng = np.random.default_rng(3)
    x = rng.normal(0, 4, size=(64, 300)).astype(np.float32)
    xb = _bf16_bits(x)
    xr = torch.from_numpy(xb.view(np.int16)).view(torch.bfloat16).float().numpy()
    a = oracle.confidence(xb, 64, 1, 300, 300, 1.3, kind=oracle.ENTROPY)
    b = oracle.confidence(xr, 64, 1, 300, 300, 1.3, kind=oracle.ENTROPY)
    assert np.array_equal(a["conf"], b["conf"]) and np.array_equal(a["argmax"], b["argmax"])


def test_stride_and_row_index():
    rng = np.random.default_rng(5)
    n, C, S = 20, 13, 16
    x = rng.normal(size=(n, S)).astype(np.float32)
    x[:, C:] = np.nan   # padding must never be read
    ri = np.array([19, 3, 3, 0, 7], np.int64)
    r = oracle.confidence(x, len(ri), 1, C, S, 0.9, row_index=ri)
    for i, row in enumerate(ri):
        p, H, am = oracle.row_stats(x[row, :C].astype(np.float64), 0.9)
        assert r["conf"][i] == p and r["argmax"][i] == am


def test_sequence_min_mean_and_correct():
    """P:423 min over tokens; MEAN (north_star); correct = all L tokens (G13)."""
    rng = np.random.default_rng(11)
    n, L, C = 6, 5, 9
    x = rng.normal(0, 2, size=(n * L, C)).astype(np.float32)
    per_tok = oracle.confidence(x, n * L, 1, C, C, 1.0)
    tok_c = per_tok["conf"].reshape(n, L)
    labels = per_tok["argmax"].copy()
    labels[7] = (labels[7] + 1) % C          # sequence 1 has one wrong token
    mn = oracle.confidence(x, n, L, C, C, 1.0, reduce=oracle.SEQ_MIN, labels=labels)
    me = oracle.confidence(x, n, L, C, C, 1.0, reduce=oracle.SEQ_MEAN, labels=labels)
    assert np.array_equal(mn["conf"], tok_c.min(axis=1))
    assert np.allclose(me["conf"], tok_c.mean(axis=1), rtol=1e-15, atol=0)
    assert np.all(mn["conf"] <= me["conf"])
    assert list(mn["correct"]) == [1, 0, 1, 1, 1, 1]
    assert np.array_equal(mn["argmax"], per_tok["argmax"])


def test_qa_min_start_end():
    """P:427-430 / S:142: start saturated, end uniform over 8 -> MAXPROB_SQ 1/64, MAXPROB 1/8."""
    start = np.array([1000, 0, 0, 0, 0, 0, 0, 0], np.float32)
    end = np.zeros(8, np.float32)
    x = np.stack([start, end])
    sq = oracle.confidence(x, 1, 2, 8, 8, 1.0, kind=oracle.MAXPROB_SQ, reduce=oracle.SEQ_MIN)
    mp = oracle.confidence(x, 1, 2, 8, 8, 1.0, kind=oracle.MAXPROB, reduce=oracle.SEQ_MIN)
    assert sq["conf"][0] == pytest.approx(1 / 64, rel=1e-15)
    assert mp["conf"][0] == pytest.approx(1 / 8, rel=1e-15)


def test_threads_do_not_change_result():
    rng = np.random.default_rng(2)
    x = rng.normal(size=(513, 77)).astype(np.float32)
    a = oracle.confidence(x, 513, 1, 77, 77, 1.0, nthreads=1)
    b = oracle.confidence(x, 513, 1, 77, 77, 1.0, nthreads=7)
    assert np.array_equal(a["conf"], b["conf"])


# ---------------------------------------------------------------------------
# NEXT-2: Top-K restricted confidence (reading G4)
# ---------------------------------------------------------------------------
def test_topk_geometric_closed_form():
    """logits (3, 2, 1, 0, ...) over a 50,000 vocabulary, top_k = 10,
    T = 1: the restricted softmax of 10 consecutive integers is a geometric
    series, p_max = (1 - e^-1) / (1 - e^-10)."""
    x = 3.0 - np.arange(50000, dtype=np.float64)
    p, H, am = oracle.row_stats(x, 1.0, top_k=10)
    want = (1 - math.exp(-1)) / (1 - math.exp(-10))
    assert p == pytest.approx(want, rel=1e-14) and am == 0
    # entropy of the truncated geometric distribution, summed independently
    q = np.array([math.exp(-i) for i in range(10)]) / sum(math.exp(-i) for i in range(10))
    assert H == pytest.approx(float(-(q * np.log(q)).sum()), rel=1e-13)


def test_topk_symmetry_and_degenerate_k():
    # top-2 restricted logits equal -> p = 1/2 (squared: 0.25)
    r = oracle.confidence(np.array([7, 7, 1, 0, -3], np.float32), 1, 1, 5, 5, 1.0,
                          kind=oracle.MAXPROB_SQ, top_k=2)
    assert r["conf"][0] == 0.25
    # K = 1: the restricted distribution is a point mass
    p, H, _ = oracle.row_stats(np.array([0.3, 2.0, -1.0]), 0.7, top_k=1)
    assert p == 1.0 and H == 0.0
    # K >= C: the full softmax
    x = np.random.default_rng(4).normal(size=37)
    for K in (37, 38, 1000):
        assert oracle.row_stats(x, 1.3, top_k=K) == oracle.row_stats(x, 1.3)


def test_topk_ties_at_the_boundary_and_masked():
    # the K largest VALUES are unique even when the K-th place is tied
    p, _, _ = oracle.row_stats(np.array([1.0, 5.0, 1.0, 1.0]), 1.0, top_k=2)
    assert p == pytest.approx(1 / (1 + math.exp(-4)), rel=1e-15)
    # -inf (masked) classes inside the top K contribute p = 0
    p, _, am = oracle.row_stats(np.array([2.0, -np.inf, 1.0, -np.inf]), 1.0, top_k=3)
    assert p == pytest.approx(1 / (1 + math.exp(-1)), rel=1e-15) and am == 0


def test_topk_library_special_case():
    """torch.topk + torch.softmax / Categorical.entropy in fp64 on random rows."""
    rng = np.random.default_rng(11)
    for _ in range(40):
        C = int(rng.integers(2, 3000))
        K = int(rng.integers(1, 40))
        T = float(rng.uniform(0.05, 5))
        x = rng.normal(scale=rng.uniform(0.1, 8), size=C)
        v = torch.topk(torch.from_numpy(x), min(K, C)).values / T
        pr = torch.softmax(v, 0)
        p, H, am = oracle.row_stats(x, T, top_k=K)
        assert p == pytest.approx(float(pr.max()), rel=1e-12)
        assert H == pytest.approx(float(torch.distributions.Categorical(probs=pr).entropy()),
                                  rel=1e-9, abs=1e-12)
        assert am == int(np.argmax(x))


def test_topk_generation_sequence_min():
    """the sequence confidence is the minimum over its tokens; each
    token restricted to its top K."""
    rng = np.random.default_rng(12)
    L, C, K = 6, 500, 8
    x = rng.normal(size=(3 * L, C)).astype(np.float32)
    r = oracle.confidence(x, 3, L, C, C, 0.9, kind=oracle.MAXPROB_SQ, reduce=oracle.SEQ_MIN,
                          top_k=K)
    for i in range(3):
        per_tok = [oracle.row_stats(x[i * L + t].astype(np.float64), 0.9, top_k=K)[0] ** 2
                   for t in range(L)]
        assert r["conf"][i] == min(per_tok)


def test_qa_hand_example_both_sides():
    """S:144 (corrected value): start (2,1,0), end (0,1,2), T = 1:
    both sides have p = e^2/(e^2+e+1); MIN = that value (squared: 0.44254...)."""
    x = np.array([[2, 1, 0], [0, 1, 2]], np.float32)
    r = oracle.confidence(x, 1, 2, 3, 3, 1.0, kind=oracle.MAXPROB_SQ, reduce=oracle.SEQ_MIN)
    e = math.e
    assert r["conf"][0] == pytest.approx((e * e / (e * e + e + 1)) ** 2, rel=1e-15)
