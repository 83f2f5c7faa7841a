"""Pins for the oracle's temperature fitting (NEXT-3; Eq. 1; clamp
range and examples S:109-117).  CPU only."""
import math

import numpy as np
import pytest
import torch

import oracle


def _data(seed, n=1500, C=12, margin=1.5, scale=1.0):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(n, C))
    y = rng.integers(0, C, size=n)
    x[np.arange(n), y] += margin
    return (x * scale).astype(np.float32), y.astype(np.int32)


def test_nll_equals_library_cross_entropy():
    x, y = _data(1)
    for T in (0.3, 1.0, 4.7):
        v, used = oracle.nll(x, y, T)
        ref = torch.nn.functional.cross_entropy(torch.from_numpy(x.astype(np.float64)) / T,
                                                torch.from_numpy(y.astype(np.int64)))
        assert used == len(y)
        assert v == pytest.approx(float(ref), rel=1e-13)


def test_two_class_closed_form():
    """Identical rows (d, 0) with a fraction q labelled 0: dNLL/dbeta = 0 at
    sigmoid(beta d) = q, so T* = d / ln(q / (1 - q))."""
    for d, q in ((3.0, 0.8), (0.5, 0.6), (7.0, 0.95)):
        n = 2000
        x = np.tile(np.array([d, 0.0], np.float32), (n, 1))
        y = np.ones(n, np.int32)
        y[: int(round(q * n))] = 0
        T = oracle.fit_temperature(x, y)
        want = d / math.log(q / (1 - q))
        assert T == pytest.approx(want, rel=1e-9)


def test_scale_equivariance_exact():
    """logits pre-multiplied by s -> T* multiplied by s (s = 8: exact in fp32)."""
    x, y = _data(2)
    t1 = oracle.fit_temperature(x, y)
    t8 = oracle.fit_temperature(x * np.float32(8), y)
    assert t8 == pytest.approx(8 * t1, rel=1e-10)


def test_clamps():
    """one record, extreme logit on the true label -> NLL decreases as
    T -> 0 -> lower clamp e^-4; every record confidently wrong -> upper clamp."""
    x = np.array([[20.0, 0.0, 0.0]], np.float32)
    assert oracle.fit_temperature(x, np.array([0], np.int32)) == pytest.approx(math.exp(-4), rel=1e-15)
    xs = np.tile(np.array([20.0, 0.0, 0.0], np.float32), (50, 1))
    assert oracle.fit_temperature(xs, np.ones(50, np.int32)) == pytest.approx(math.exp(4), rel=1e-15)


def test_minimum_against_a_fine_grid_and_t1():
    """the fitted loss is never worse than T = 1; and no point of a
    2,000-point log grid over the clamp range beats it."""
    for seed, scale in ((3, 1.0), (4, 0.2), (5, 6.0)):
        x, y = _data(seed, scale=scale)
        T = oracle.fit_temperature(x, y)
        best = oracle.nll(x, y, T)[0]
        grid = np.exp(np.linspace(-4, 4, 2000))
        vals = [oracle.nll(x, y, t)[0] for t in grid[::20]]
        assert best <= min(vals) + 1e-12
        assert best <= oracle.nll(x, y, 1.0)[0] + 1e-15
        # the interior optimum has a vanishing derivative (central difference in beta)
        b, h = 1.0 / T, 1e-4 / T
        dl = (oracle.nll(x, y, 1.0 / (b + h))[0] - oracle.nll(x, y, 1.0 / (b - h))[0]) / (2 * h)
        assert abs(dl) < 1e-7


def test_masked_and_invalid_rows():
    x, y = _data(6, n=200)
    x2 = x.copy()
    x2[:, 3] = -np.inf                      # a masked class everywhere (label never 3)
    y2 = np.where(y == 3, 4, y).astype(np.int32)
    v, used = oracle.nll(x2, y2, 1.0)
    ref = torch.nn.functional.cross_entropy(torch.from_numpy(np.delete(x2, 3, 1).astype(np.float64)),
                                            torch.from_numpy(np.where(y2 > 3, y2 - 1, y2).astype(np.int64)))
    assert used == 200 and v == pytest.approx(float(ref), rel=1e-13)
    x3 = x.copy()
    x3[0, 0] = np.nan                       # invalid rows are skipped
    assert oracle.nll(x3, y, 1.0)[1] == 199
