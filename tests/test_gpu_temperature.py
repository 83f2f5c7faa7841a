"""GPU parity of NEXT-3, temperature fitting (Eq. 1; clamp range
S:112): hs_fit_temperature vs the fp64 oracle (oracle.fit_temperature /
oracle.nll) on the same seeded logits.

Tolerance: the GPU sums each row in fp32 (ex2.approx, exact
x - m) and across rows in fp64, and stops when a Newton step in beta = 1/T is
below 2^-21 relative; its fitted T must lie within 1e-5 relative of the
oracle's minimiser, and -- what the fit is for -- the oracle's NLL at the GPU's
T must exceed the oracle's minimum by at most 1e-9 (relative: the objective is
flat at the minimum, so this is much tighter than the T tolerance).  The GPU's
reported NLL must equal the oracle's NLL at the GPU's T within 1e-5 relative.
Used-row counts are exact; clamp ends are returned exactly."""
import math

import numpy as np
import pytest
import torch

import oracle
from workload import synth

pytestmark = pytest.mark.gpu

T_REL = 1e-5
NLL_EXCESS = 1e-9
NLL_REL = 1e-5


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def dev():
    return torch.device("cuda:0")


def to_dev(x: np.ndarray, dtype: str, stride: int | None = None) -> torch.Tensor:
    """fp32 values (bf16-representable when dtype == 'bf16') or raw bf16 bits -> CUDA [rows, stride]."""
    rows, C = x.shape
    stride = stride or C
    if dtype == "bf16":
        bits = x if x.dtype == np.uint16 else _bf16_bits(x)
        t = torch.zeros(rows, stride, dtype=torch.int16)
        t[:, :C] = torch.from_numpy(bits.view(np.int16))
        return t.to(dev()).view(torch.bfloat16)
    t = torch.zeros(rows, stride, dtype=torch.float32)
    t[:, :C] = torch.from_numpy(x)
    return t.to(dev())


def _bf16_bits(x32: np.ndarray) -> np.ndarray:
    """fp32 -> bf16 bits, round to nearest even (finite inputs) / exact for inf, nan."""
    u = np.ascontiguousarray(x32, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    special = ~np.isfinite(x32)
    r[special] = (u[special] >> 16).astype(np.uint16)
    return r


def host_rows(t: torch.Tensor, C: int) -> np.ndarray:
    if t.dtype == torch.bfloat16:
        return np.ascontiguousarray(t.view(torch.int16).cpu().numpy().view(np.uint16)[:, :C])
    return np.ascontiguousarray(t.cpu().numpy()[:, :C])


def fit(hs, xs, labels, C=None, **kw):
    status = torch.zeros(1, dtype=torch.int32, device=dev())
    lab = torch.from_numpy(np.ascontiguousarray(labels, np.int32)).to(dev())
    r = hs.fit_temperature(xs, lab, n_classes=C, status=status, **kw)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in r.items()}
    out["status"] = int(status.item())
    return out


def check_against_oracle(hs, xs, labels, C, t_lo=None, t_hi=None):
    kw = {}
    if t_lo is not None:
        kw = dict(t_lo=t_lo, t_hi=t_hi)
    g = fit(hs, xs, labels, C, **kw)
    for b, x in enumerate(xs):
        rows = host_rows(x, C)
        ora_kw = {} if t_lo is None else dict(t_lo=t_lo, t_hi=t_hi)
        t_o = oracle.fit_temperature(rows, labels, n_classes=C, **ora_kw)
        t_g = float(g["T"][b])
        assert abs(t_g - t_o) <= T_REL * t_o, (b, t_g, t_o, g["passes"][b])
        best, used = oracle.nll(rows, labels, t_o, n_classes=C)
        at_g, _ = oracle.nll(rows, labels, t_g, n_classes=C)
        assert int(g["used"][b]) == used
        assert at_g - best <= NLL_EXCESS * abs(best), (b, at_g, best)
        assert abs(g["nll"][b] - at_g) <= NLL_REL * abs(at_g), (b, g["nll"][b], at_g)
        assert g["status"] & 2 == 0
    return g


def test_fit_c2_validation_stages(hs):
    """The C2 validation workload (5 ViT stages, 1,000 classes, bf16, the
    generator's logits), reduced to 3,000 samples, all stages in one launch."""
    fam = synth.FAMILIES["c2"]
    n = 3000
    vids = np.arange(n, dtype=np.int64) + synth.VAL_ID_BASE
    labels = synth.labels_np(fam.seed, vids, 1, fam.C).reshape(-1)
    xs = [to_dev(synth.fam_logits_np(fam, k, vids, "bf16", L=1, C=fam.C), "bf16")
          for k in range(fam.K)]
    g = check_against_oracle(hs, xs, labels, fam.C)
    assert (g["passes"] <= 12).all(), g["passes"]


def _gauss_rows(seed, n, C, margin=2.0, scale=1.5):
    rng = np.random.default_rng(seed)
    x = rng.normal(size=(n, C)).astype(np.float32) * np.float32(scale)
    y = rng.integers(0, C, size=n).astype(np.int32)
    # the label wins with probability ~0.7, else a random class gets the margin
    win = np.where(rng.random(n) < 0.7, y, rng.integers(0, C, size=n))
    x[np.arange(n), win] += np.float32(margin)
    return x, y


@pytest.mark.parametrize("C", [2, 7, 129, 1000, 4099, 32128])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_fit_shapes(hs, C, dtype):
    """Every lanes-per-row instantiation, ragged last vectors, padded strides."""
    n = max(40, min(1500, 2_000_000 // C))
    xs = []
    for k in range(2):
        x, y = _gauss_rows(100 + k + C, n, C, margin=1.0 + k, scale=0.5 + k)
        if dtype == "bf16":
            x = _bf16_bits(x).view(np.uint16)
        ve = 8 if dtype == "bf16" else 4
        xs.append(to_dev(x, dtype, stride=(C + ve - 1) // ve * ve + ve * (C % 3)))
    _, y = _gauss_rows(100 + C, n, C)
    check_against_oracle(hs, xs, y, C)


def test_fit_two_class_closed_form(hs):
    """Rows (d, 0), a fraction q labelled 0: T* = d / ln(q / (1 - q))."""
    for d, q in ((3.0, 0.8), (0.5, 0.6), (7.0, 0.95)):
        n = 2000
        x = np.tile(np.array([d, 0.0], np.float32), (n, 1))
        y = np.ones(n, np.int32)
        y[: int(round(q * n))] = 0
        g = fit(hs, [to_dev(x, "fp32", stride=4)], y, 2)
        want = d / math.log(q / (1 - q))
        assert abs(g["T"][0] - want) <= T_REL * want, (g["T"][0], want)


def test_fit_clamps_exact(hs):
    """a confidently right record -> T = t_lo exactly; every record
    confidently wrong -> T = t_hi exactly."""
    x = np.tile(np.array([20.0, 0.0, 0.0, 0.0], np.float32), (64, 1))
    g = fit(hs, [to_dev(x, "fp32"), to_dev(x, "fp32")], np.zeros(64, np.int32), 3)
    assert g["T"][0] == np.float32(math.exp(-4)) and g["T"][1] == np.float32(math.exp(-4))
    g = fit(hs, [to_dev(x, "fp32")], np.ones(64, np.int32), 3)
    assert g["T"][0] == np.float32(math.exp(4))
    g = fit(hs, [to_dev(x, "fp32")], np.ones(64, np.int32), 3, t_lo=0.5, t_hi=2.0)
    assert g["T"][0] == np.float32(2.0)
    assert g["passes"][0] <= 3


def test_fit_scale_equivariance(hs):
    """logits x 8 -> T x 8 (x 8 is exact in fp32 and bf16)."""
    x, y = _gauss_rows(7, 1000, 100)
    g1 = fit(hs, [to_dev(x, "fp32")], y, 100)
    g8 = fit(hs, [to_dev(x * np.float32(8), "fp32")], y, 100)
    assert abs(g8["T"][0] - 8 * g1["T"][0]) <= 2 * T_REL * 8 * g1["T"][0]


def test_fit_invalid_and_masked_rows(hs):
    x, y = _gauss_rows(8, 600, 64)
    x[:, 5] = -np.inf                         # masked class
    y = np.where(y == 5, 6, y).astype(np.int32)
    x[0, 0] = np.nan                          # invalid: NaN
    x[1, :] = -np.inf                         # invalid: all -inf
    x[2, 1] = np.inf                          # invalid: +inf
    y[3] = 5                                  # label logit -inf: unused, not an error
    for dtype in ("fp32", "bf16"):
        xx = x if dtype == "fp32" else _bf16_bits(x).view(np.uint16)
        g = check_against_oracle(hs, [to_dev(xx, dtype)], y, 64)
        assert g["used"][0] == 596
        assert g["status"] & 1


def test_fit_empty_and_deterministic(hs):
    x, y = _gauss_rows(9, 5000, 1000)
    xs = [to_dev(_bf16_bits(x).view(np.uint16), "bf16")]
    a = fit(hs, xs, y, 1000)
    b = fit(hs, xs, y, 1000)
    assert a["T"].tobytes() == b["T"].tobytes() and a["nll"].tobytes() == b["nll"].tobytes()
    e = fit(hs, [xs[0][:0]], np.zeros(0, np.int32), 1000)
    assert np.isnan(e["T"][0]) and e["used"][0] == 0 and e["status"] == 0


def test_fit_pass_budget(hs):
    """max_passes = 1: not converged -> status bit 2 and the swept T = 1."""
    x, y = _gauss_rows(10, 2000, 50, margin=4.0, scale=0.3)
    g = fit(hs, [to_dev(x, "fp32", stride=52)], y, 50, max_passes=1)
    assert g["passes"][0] == 1 and g["status"] & 2 and g["T"][0] == 1.0
    nll1, _ = oracle.nll(x, y, 1.0)
    assert abs(g["nll"][0] - nll1) <= NLL_REL * nll1


@pytest.mark.parametrize("dtype,C", [("bf16", 128), ("fp32", 64)])
def test_fit_warm_start_path(hs, dtype, C):
    """n >= 32,768 rows of <= 2 KB: the fit starts with Newton sweeps over every
    16th row before the full sweeps; the result is still the full objective's
    minimiser (same tolerances), for three models with different optima."""
    n = 40000
    xs, ys = [], None
    for k in range(3):
        x, y = _gauss_rows(200 + k, n, C, margin=1.0 + 1.5 * k, scale=0.4 + 0.6 * k)
        if ys is None:
            ys = y
        if dtype == "bf16":
            x = _bf16_bits(x).view(np.uint16)
        xs.append(to_dev(x, dtype))
    g = check_against_oracle(hs, xs, ys, C)
    assert (g["passes"] <= 4).all(), g["passes"]
