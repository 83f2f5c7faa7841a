"""The fused cascade step (K1 with the threshold test and the stable compaction
in its row epilogue, one launch per stage) against the two-launch step (K1
then K3, the default) and against the oracle.  The fused step is opt-in
(HS_FUSE=1): measured slower than the two launches on C2.

Both paths compute every confidence with the same row reduction, so every
output -- accepted ids / confidences / argmaxes, the deferred list (the next
stage's batch), the payload gather and the counts -- must agree bit
for bit, at tile edges (1, 15, 16, 17 rows; tiles of up to 1,024 chunks), with
device-resident counts and thresholds, gathered rows, NaN rows, thresholds 0 /
1 / +inf, the last stage, and over repeated launches on one workspace (the
tile counters alternate between two banks by launch epoch; each launch zeroes
the bank of the next)."""
import numpy as np
import pytest
import torch

import oracle
from workload import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def dev():
    return torch.device("cuda:0")


def rand_logits(n, C, dtype, seed, nan_rows=0):
    g = torch.Generator().manual_seed(seed)
    x = torch.randn(n, C, generator=g) * 3.0
    # a spread of confidences: scale some rows up (confident) and ties in a few
    scale = torch.rand(n, 1, generator=g) * 4.0
    x = x * scale
    if n > 8:
        x[3, :] = 0.0                         # uniform row: conf 1/C, argmax 0
        x[5, 1] = x[5].max() + 1.0
        x[5, 3] = x[5, 1]                     # tie: lowest index wins
    for r in range(min(nan_rows, n)):
        x[(r * 7919) % n, r % C] = float("nan")
    x = x.to(torch.bfloat16 if dtype == "bf16" else torch.float32)
    return x.to(dev())


def step(hs, monkeypatch, fused, x, thr, *, stage=0, K=3, n=None, ids=None, d_n=None, row_index=None,
         payload=None, P=0, ws=None, T=1.0, kind="maxprob"):
    monkeypatch.setenv("HS_FUSE", "1" if fused else "0")
    n = x.shape[0] if n is None else n
    status = torch.zeros(1, dtype=torch.int32, device=dev())
    out = hs.cascade_step(stage, K, x, thr, n=n, temperature=T, kind=kind, ids=ids, d_n=d_n,
                          row_index=row_index, payload=payload, payload_row_bytes=P, ws=ws,
                          status=status)
    torch.cuda.synchronize()
    return out


def assert_same(a, b, P=0):
    ca, cb = a["counts"].cpu().tolist(), b["counts"].cpu().tolist()
    assert ca == cb, (ca, cb)
    na, nd = ca
    for key, m in (("acc_ids", na), ("acc_pred", na), ("next_ids", nd)):
        assert torch.equal(a[key][:m], b[key][:m]), key
    # confidences bit for bit (NaN included)
    assert torch.equal(a["acc_conf"][:na].view(torch.int32), b["acc_conf"][:na].view(torch.int32))
    if P:
        assert torch.equal(a["next_payload"][:nd * P], b["next_payload"][:nd * P])


@pytest.mark.parametrize("C,dtype", [(1000, "bf16"), (64, "bf16"), (500, "f32"), (100, "f32"), (8, "bf16")])
@pytest.mark.parametrize("n", [1, 15, 16, 17, 1023, 16 * 1024 + 5, 70001])
def test_fused_equals_two_launch(hs, monkeypatch, C, dtype, n):
    x = rand_logits(n, C, dtype, seed=n * 31 + C, nan_rows=3)
    for thr in (0.0, 0.35, 1.0, float("inf")):
        a = step(hs, monkeypatch, True, x, thr)
        b = step(hs, monkeypatch, False, x, thr)
        assert_same(a, b)
    # the last stage accepts every row, NaN confidences included
    a = step(hs, monkeypatch, True, x, 0.5, stage=2)
    b = step(hs, monkeypatch, False, x, 0.5, stage=2)
    assert_same(a, b)
    assert a["counts"].cpu().tolist() == [n, 0]


@pytest.mark.parametrize("n", [300, 40000, 262144])
def test_fused_ids_payload_device_count(hs, monkeypatch, n):
    """Later-stage shape: ids of the batch, a 48-B payload gathered for the
    deferred rows, the live count and the threshold on the device (capacity-
    sized buffers, count smaller than the capacity; also a count of 0)."""
    C = 1000
    cap = n + 333
    x = rand_logits(cap, C, "bf16", seed=n)
    g = torch.Generator().manual_seed(n + 1)
    ids = (torch.randperm(10 * cap, generator=g)[:cap]).to(torch.int64).to(dev())
    P = 48
    payload = torch.randint(0, 255, (cap, P), generator=g, dtype=torch.uint8).to(dev())
    thr = torch.tensor([0.41], dtype=torch.float32, device=dev())
    for live in (n, 0, 1):
        d_n = torch.tensor([live], dtype=torch.int64, device=dev())
        a = step(hs, monkeypatch, True, x, thr, stage=1, n=cap, ids=ids, d_n=d_n, payload=payload, P=P)
        b = step(hs, monkeypatch, False, x, thr, stage=1, n=cap, ids=ids, d_n=d_n, payload=payload, P=P)
        assert_same(a, b, P)
        assert sum(a["counts"].cpu().tolist()) == live


def test_fused_row_index_entropy(hs, monkeypatch):
    """Gathered rows (row_index: the by-id layout) and the entropy confidence."""
    n, C = 50000, 1000
    x = rand_logits(3 * n, C, "bf16", seed=7)
    g = torch.Generator().manual_seed(8)
    ri = torch.randperm(3 * n, generator=g)[:n].to(torch.int64).to(dev())
    for kind in ("maxprob", "entropy"):
        a = step(hs, monkeypatch, True, x, 0.3, n=n, ids=ri, row_index=ri, kind=kind, T=1.7)
        b = step(hs, monkeypatch, False, x, 0.3, n=n, ids=ri, row_index=ri, kind=kind, T=1.7)
        assert_same(a, b)


def test_fused_repeated_launches_one_workspace(hs, monkeypatch):
    """Many launches of different sizes and thresholds on one workspace (tile
    counter banks alternating by epoch), eagerly and from a CUDA graph."""
    C, cap = 1000, 200000
    x = rand_logits(cap, C, "bf16", seed=11)
    ws = hs.workspace(hs.lib().hs_cascade_step_workspace(cap, 1), dev())
    sizes = [cap, 17, 150001, 1, 99999, cap]
    thrs = [0.2, 0.9, 0.5, 0.0, 0.33, 0.61]
    refs = []
    for live, t in zip(sizes, thrs):
        d_n = torch.tensor([live], dtype=torch.int64, device=dev())
        b = step(hs, monkeypatch, False, x, t, stage=1, n=cap, d_n=d_n)
        refs.append({k: v.clone() for k, v in b.items()})
    for rep in range(3):
        for (live, t), b in zip(zip(sizes, thrs), refs):
            d_n = torch.tensor([live], dtype=torch.int64, device=dev())
            a = step(hs, monkeypatch, True, x, t, stage=1, n=cap, d_n=d_n, ws=ws)
            assert_same(a, b)
    # graph replay: a captured sequence of fused steps on the shared workspace
    monkeypatch.setenv("HS_FUSE", "1")
    d_ns = [torch.tensor([live], dtype=torch.int64, device=dev()) for live in sizes]
    d_ts = [torch.tensor([t], dtype=torch.float32, device=dev()) for t in thrs]
    outs = [None] * len(sizes)
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        def seq():
            for i in range(len(sizes)):
                outs[i] = hs.cascade_step(1, 3, x, d_ts[i], n=cap, d_n=d_ns[i], ws=ws, out=outs[i], stream=s)
        seq()
        s.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            seq()
        for _ in range(4):
            g.replay()
    torch.cuda.synchronize()
    for a, b in zip(outs, refs):
        assert_same(a, b)


def test_fused_cascade_vs_oracle_production_shape(hs, monkeypatch):
    """C2 rows (1,000 bf16 classes) through 3 fused stages vs the oracle's
    cascade (D4), near-threshold requests counted and excluded."""
    monkeypatch.setenv("HS_FUSE", "1")
    fam = synth.FAMILIES["c2"]
    n, K = 30011, 3
    gen_ids = np.arange(n, dtype=np.int64) + 12345
    logits, conf_o = [], []
    for k in range(K):
        bits = synth.fam_logits_np(fam, k, gen_ids, "bf16", L=1, C=fam.C)
        t = torch.from_numpy(bits.view(np.int16)).to(dev()).view(torch.bfloat16)
        logits.append(t)
        conf_o.append(oracle.confidence(bits, n, 1, fam.C, fam.C, fam.temps[k])["conf"])
    conf_o = np.stack(conf_o)
    t = [float(np.float32(np.quantile(conf_o[0], 0.4))), float(np.float32(np.quantile(conf_o[1], 0.5))), 0.0]
    casc = hs.Cascade(n, [hs.StageSpec(fam.C, fam.temps[k], 1, "maxprob", "none") for k in range(K)], dev())
    casc.route(logits, t, by_id=True)          # stage k reads request r's row r (row_index)
    res = casc.results()
    tt = np.array(t, np.float64)
    stage_of = oracle.cascade(conf_o, tt)
    lists = oracle.stage_lists(stage_of, K)
    near = np.zeros(n, bool)
    for k in range(K - 1):
        near |= (stage_of >= k) & (np.abs(conf_o[k] - tt[k]) <= 1e-5 * tt[k])
    print(f"near-threshold requests: {int(near.sum())} of {n}")
    for k in range(K):
        got = res[k]["ids"].numpy()
        want = lists[k][1]
        assert np.array_equal(got[~near[got]], want[~near[want]])


# ---------------------------------------------------------------------------
# The last stage without a compaction: it accepts every row in order, so K1
# writes the accepted lists and the counts itself (HS_LAST_K3=1: K1 then K3)
# ---------------------------------------------------------------------------
def last_step(hs, monkeypatch, direct, x, *, n=None, ids=None, d_n=None, row_index=None, top_k=0, kind="maxprob"):
    monkeypatch.setenv("HS_LAST_K3", "0" if direct else "1")
    n = x.shape[0] if n is None else n
    status = torch.zeros(1, dtype=torch.int32, device=dev())
    out = hs.cascade_step(2, 3, x, 0.5, n=n, ids=ids, d_n=d_n, row_index=row_index, status=status,
                          kind=kind, top_k=top_k, temperature=1.3)
    torch.cuda.synchronize()
    return out


@pytest.mark.parametrize("C,dtype,n", [(1000, "bf16", 70001), (1000, "f32", 4097), (64, "bf16", 17),
                                       (32128, "bf16", 300), (128256, "bf16", 40), (2000, "f32", 1)])
def test_last_stage_direct_equals_compaction(hs, monkeypatch, C, dtype, n):
    """Every K1 path (cp.async rows, register rows, warp per vocabulary row,
    split rows for small batches): the same accepted lists and counts as K1
    then K3, with ids given or the identity, a device count (also 0), gathered
    rows, and the entropy kind."""
    x = rand_logits(n, C, dtype, seed=C + n, nan_rows=2)
    cap = n
    g = torch.Generator().manual_seed(n)
    ids = torch.randperm(5 * cap, generator=g)[:cap].to(torch.int64).to(dev())
    for kw in ({}, {"ids": ids}, {"ids": ids, "row_index": torch.arange(n - 1, -1, -1, device=dev())},
               {"kind": "entropy"}):
        a = last_step(hs, monkeypatch, True, x, **kw)
        b = last_step(hs, monkeypatch, False, x, **kw)
        assert_same(a, b)
        assert a["counts"].cpu().tolist() == [n, 0]
    for live in (n // 2, 0):
        d_n = torch.tensor([live], dtype=torch.int64, device=dev())
        a = last_step(hs, monkeypatch, True, x, n=cap, ids=ids, d_n=d_n)
        b = last_step(hs, monkeypatch, False, x, n=cap, ids=ids, d_n=d_n)
        assert_same(a, b)
        assert a["counts"].cpu().tolist() == [live, 0]


def test_last_stage_direct_topk(hs, monkeypatch):
    x = rand_logits(3000, 32128, "bf16", seed=5)
    a = last_step(hs, monkeypatch, True, x, top_k=10)
    b = last_step(hs, monkeypatch, False, x, top_k=10)
    assert_same(a, b)


@pytest.mark.parametrize("C,dtype", [(1000, "bf16"), (200, "f32")])
def test_logits_capacity_flag_early_rows(hs, monkeypatch, C, dtype):
    """HS_STEP_LOGITS_CAPACITY (set by the binding when the logits memory covers
    the capacity): dense rows are read before the device count is known; the
    cascade step equals the one on an exact-sized copy of the live rows (flag
    off), for several live counts, middle and last stage."""
    monkeypatch.setenv("HS_FUSE", "0")
    cap = 100003
    x = rand_logits(cap, C, dtype, seed=C)
    g = torch.Generator().manual_seed(3)
    ids = torch.randperm(4 * cap, generator=g)[:cap].to(torch.int64).to(dev())
    assert hs._rows_capacity_flag(x, cap, None) == hs.HS_STEP_LOGITS_CAPACITY
    for live in (cap, 65537, 17, 1, 0):
        d_n = torch.tensor([live], dtype=torch.int64, device=dev())
        exact = x[: max(live, 1)].clone()
        assert hs._rows_capacity_flag(exact, cap, None) == (hs.HS_STEP_LOGITS_CAPACITY if live >= cap else 0)
        for stage in (1, 2):
            a = hs.cascade_step(stage, 3, x, 0.4, n=cap, ids=ids, d_n=d_n)
            b = hs.cascade_step(stage, 3, exact, 0.4, n=cap, ids=ids, d_n=d_n)
            torch.cuda.synchronize()
            assert_same(a, b)
            assert sum(a["counts"].cpu().tolist()) == live
