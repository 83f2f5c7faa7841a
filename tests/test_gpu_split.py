"""GPU parity of K1e, the split-row confidence path that hs_cascade_step uses
for small batches of long rows (routing latency, Fig. 8): every
row is cut into segments reduced by different warps and merged by the last
one to arrive.  Same bar as K1 (test_gpu_parity.py): confidences within 1e-5
relative of the fp64 oracle, argmax exact (lowest index on ties, also across
segments), NaN pattern exact; results bitwise repeatable and the per-row
arrival counters re-armed between calls."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
REL = 1e-5


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def dev():
    return torch.device("cuda:0")


def _bf16_bits(x32):
    u = np.ascontiguousarray(x32, np.float32).view(np.uint32).astype(np.uint64)
    r = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16).astype(np.uint16)
    sp = ~np.isfinite(x32)
    r[sp] = (u[sp] >> 16).astype(np.uint16)
    return r


def run_step(hs, rows_np, dtype, C, T, kind, ws=None):
    """Last-stage cascade step (accepts every row): acc_conf / acc_pred in order."""
    n = rows_np.shape[0]
    if dtype == "bf16":
        bits = _bf16_bits(rows_np)
        x = torch.from_numpy(bits.view(np.int16)).to(dev()).view(torch.bfloat16)
        host = bits
    else:
        x = torch.from_numpy(np.ascontiguousarray(rows_np, np.float32)).to(dev())
        host = np.ascontiguousarray(rows_np, np.float32)
    st = torch.zeros(1, dtype=torch.int32, device=dev())
    out = hs.cascade_step(0, 1, x, 0.0, n=n, n_classes=C, temperature=T, kind=kind, ws=ws, status=st)
    torch.cuda.synchronize()
    assert int(out["counts"][0]) == n
    return out["acc_conf"][:n].cpu().numpy(), out["acc_pred"][:n].cpu().numpy(), host, int(st.item())


def check(hs, rows_np, dtype, C, T, kind, ws=None):
    conf, am, host, st = run_step(hs, rows_np, dtype, C, T, kind, ws)
    ref = oracle.confidence(host, rows_np.shape[0], 1, C, C, T, kind=kind)
    nan_o = np.isnan(ref["conf"])
    assert np.array_equal(np.isnan(conf), nan_o)
    if (~nan_o).any():
        err = np.abs(conf[~nan_o] - ref["conf"][~nan_o]) / ref["conf"][~nan_o]
        assert err.max() <= REL, err.max()
    assert np.array_equal(am, ref["argmax"])
    return conf, am, st


@pytest.mark.parametrize("dtype,C,n,kind,T", [
    ("bf16", 32128, 1, 0, 1.0), ("bf16", 32128, 3, 0, 0.7), ("bf16", 32128, 64, 1, 1.0),
    ("bf16", 128256, 1, 2, 1.0), ("bf16", 128256, 17, 2, 2.0), ("fp32", 262144, 1, 0, 1.0),
    ("fp32", 262144, 2, 2, 0.5), ("fp32", 5000, 7, 0, 1.0), ("bf16", 4104, 1, 2, 1.0),
    ("bf16", 32128, 2048, 0, 1.0)])
def test_split_rows_vs_oracle(hs, dtype, C, n, kind, T):
    rng = np.random.default_rng(C + n + kind)
    x = (rng.normal(size=(n, C)) * 2.0).astype(np.float32)
    win = rng.integers(0, C, size=n)
    x[np.arange(n), win] += 6.0
    check(hs, x, dtype, C, T, kind)


def test_split_adversarial_rows(hs):
    C = 32128
    rng = np.random.default_rng(5)
    x = rng.normal(size=(8, C)).astype(np.float32)
    x[0, [100, 20000, 31000]] = 9.0          # the max tied in three segments: lowest index wins
    x[1, -1] = np.nan                        # NaN in the last segment
    x[2, :] = -np.inf                        # all -inf: invalid
    x[3, :16000] = -np.inf                   # masked first half
    x[4, 30000] = np.inf                     # +inf: invalid
    x[5, :] = 1e-40                          # subnormal max everywhere: argmax 0
    x[6, 31999] = 50.0                       # max in the last vector of the last segment
    x[7, 0] = 50.0                           # max in the first element
    for dtype in ("bf16", "fp32"):
        for kind in (0, 2):
            conf, am, st = check(hs, x, dtype, C, 1.0, kind)
            assert st & 1
            assert am[0] == 100 and am[6] == 31999 and am[7] == 0 and am[5] == 0


def test_split_repeatable_and_rearmed(hs):
    C = 128256
    rng = np.random.default_rng(9)
    x = rng.normal(size=(5, C)).astype(np.float32)
    ws = hs.workspace(hs.lib().hs_cascade_step_workspace(5, 1), dev())
    a = run_step(hs, x, "bf16", C, 1.0, 2, ws)
    b = run_step(hs, x, "bf16", C, 1.0, 2, ws)
    assert a[0].tobytes() == b[0].tobytes() and np.array_equal(a[1], b[1])
    # different rows through the same workspace: the arrival counters were re-armed
    for seed in (10, 11, 12):
        y = np.random.default_rng(seed).normal(size=(5, C)).astype(np.float32) * 3
        check(hs, y, "bf16", C, 1.0, 2, ws)


@pytest.mark.parametrize("reduce", [1, 2])
def test_split_rows_in_sequences(hs, reduce):
    """Token rows of a few T5-like sequences (4 x 64 tokens of 32,128 classes:
    256 rows, split path) reduced to sequence confidences (MIN / MEAN)
    with their argmaxes, through a last-stage cascade step, vs the oracle."""
    n, L, C = 4, 64, 32128
    rng = np.random.default_rng(31 + reduce)
    x = (rng.normal(size=(n * L, C)) * 1.5).astype(np.float32)
    x[np.arange(n * L), rng.integers(0, C, size=n * L)] += 7.0
    bits = _bf16_bits(x)
    xt = torch.from_numpy(bits.view(np.int16)).to(dev()).view(torch.bfloat16)
    out = hs.cascade_step(0, 1, xt, 0.0, n=n, seq_len=L, n_classes=C, temperature=1.0, reduce=reduce)
    torch.cuda.synchronize()
    ref = oracle.confidence(bits, n, L, C, C, 1.0, reduce=reduce)
    conf = out["acc_conf"][:n].cpu().numpy()
    assert np.max(np.abs(conf - ref["conf"]) / ref["conf"]) <= REL
    assert np.array_equal(out["acc_pred"][: n * L].cpu().numpy(), ref["argmax"])


def test_split_through_hs_confidence(hs):
    """hs_confidence with its full workspace (not zero-filled: torch.empty) takes
    the split-row path for a few long rows; results vs the oracle, repeatable."""
    C = 128256
    rng = np.random.default_rng(41)
    for n, kind in ((1, 2), (3, 0), (17, 1)):
        x = rng.normal(size=(n, C)).astype(np.float32) * 2
        bits = _bf16_bits(x)
        xt = torch.from_numpy(bits.view(np.int16)).to(dev()).view(torch.bfloat16)
        ws = torch.full((hs.lib().hs_confidence_workspace(n, 1),), 0xAB, dtype=torch.uint8, device=dev())
        for _ in range(2):
            r = hs.confidence(xt, temperature=1.3, kind=kind, ws=ws)
            torch.cuda.synchronize()
            ref = oracle.confidence(bits, n, 1, C, C, 1.3, kind=kind)
            assert np.max(np.abs(r["conf"].cpu().numpy() - ref["conf"]) / ref["conf"]) <= REL
            assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"])
