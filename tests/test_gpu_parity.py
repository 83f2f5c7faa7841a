"""GPU parity: the CUDA path (through the C-ABI) vs the fp64 CPU oracle on the
same seeded inputs.  Tolerances (north_star): confidences within 1e-5 relative;
argmax, correct bits, routing decisions, compacted lists and calibrated
threshold indices bit-exact, except requests whose oracle confidence lies within
1e-5 (relative) of a threshold, which are counted and excluded."""
import math

import numpy as np
import pytest
import torch

import oracle
import workload
from workload import synth

pytestmark = pytest.mark.gpu

REL = 1e-5


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def dev():
    return torch.device("cuda:0")


def to_dev_bits(bits: np.ndarray, dtype: str, stride: int | None = None) -> torch.Tensor:
    """numpy logits (raw bf16 bits or fp32) [rows, C] -> CUDA tensor [rows, stride]."""
    rows, C = bits.shape
    stride = stride or C
    if dtype == "bf16":
        t = torch.zeros(rows, stride, dtype=torch.int16)
        t[:, :C] = torch.from_numpy(bits.view(np.int16))
        return t.to(dev()).view(torch.bfloat16)
    t = torch.zeros(rows, stride, dtype=torch.float32)
    t[:, :C] = torch.from_numpy(bits)
    return t.to(dev())


def host_bits(x: torch.Tensor) -> np.ndarray:
    if x.dtype == torch.bfloat16:
        return x.view(torch.int16).cpu().numpy().view(np.uint16)
    return x.cpu().numpy()


def assert_conf_close(g: np.ndarray, o: np.ndarray):
    g = g.astype(np.float64)
    nan_o = np.isnan(o)
    assert np.array_equal(np.isnan(g), nan_o), "NaN pattern differs"
    err = np.abs(g[~nan_o] - o[~nan_o]) / np.maximum(np.abs(o[~nan_o]), 1e-300)
    assert err.size == 0 or err.max() <= REL, f"max rel err {err.max():.3e}"
    return 0.0 if err.size == 0 else float(err.max())


def run_conf(hs, x, fam_like, n, L, C, T, kind, reduce, labels=None, row_index=None):
    status = torch.zeros(1, dtype=torch.int32, device=dev())
    lab = None if labels is None else torch.from_numpy(np.ascontiguousarray(labels, np.int32)).to(dev())
    ri = None if row_index is None else torch.from_numpy(np.asarray(row_index, np.int64)).to(dev())
    r = hs.confidence(x, n=n, seq_len=L, n_classes=C, temperature=T, kind=kind, reduce=reduce,
                      labels=lab, row_index=ri, status=status)
    torch.cuda.synchronize()
    return r, int(status.item())


def check_family(hs, fam, n, kinds=None, stride_pad=0, T=None):
    ids = np.arange(n, dtype=np.int64) * 7 + 3
    L, C = fam.L, fam.C
    bits = synth.fam_logits_np(fam, 0, ids, fam.dtype, L=L, C=C)
    lab = synth.labels_np(fam.seed, ids, L, C).reshape(-1)
    eb = 2 if fam.dtype == "bf16" else 4
    stride = C + stride_pad
    x = to_dev_bits(bits, fam.dtype, stride)
    worst = 0.0
    for kind in (kinds or [fam.kind]):
        T_ = T or fam.temps[0]
        r, st = run_conf(hs, x, fam, n, L, C, T_, kind, fam.reduce, labels=lab)
        ref = oracle.confidence(host_bits(x), n, L, C, stride, T_, kind=kind, reduce=fam.reduce,
                                labels=lab)
        assert st == 0
        worst = max(worst, assert_conf_close(r["conf"].cpu().numpy(), ref["conf"]))
        assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"])
        assert np.array_equal(r["correct"].cpu().numpy(), ref["correct"])
    return worst


# ---------------------------------------------------------------------------
# K1/K2 confidence
# ---------------------------------------------------------------------------
def test_conf_c1_full_fp32(hs):
    fam = synth.FAMILIES["c1"]
    check_family(hs, fam, fam.n, kinds=[0, 1, 2])


def test_conf_c2_bf16_all_kinds(hs):
    check_family(hs, synth.FAMILIES["c2"], 9000, kinds=[0, 1, 2])


@pytest.mark.parametrize("C", [2, 3, 8, 17, 255, 256, 257, 1000, 2047, 2048, 4096, 4100, 9000,
                               32128])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_conf_class_counts_and_tails(hs, C, dtype):
    """Every launch shape (warp-per-row NV=1..16, CTA-per-row) and ragged last vectors."""
    ve = 8 if dtype == "bf16" else 4
    pad = (-C) % ve
    fam = synth.Family("t", 0, C, 1, dtype, (0.6,), (1.0,), 0, 0, 1)
    n = 300 if C <= 4096 else 40
    check_family(hs, fam, n, kinds=[0, 2], stride_pad=pad + (ve if C % 5 == 0 else 0))


def test_conf_t5_sequences_min_mean(hs):
    fam = synth.scaled(synth.FAMILIES["c3"], L=6)
    for reduce in (1, 2):
        f = synth.dataclasses.replace(fam, reduce=reduce)
        check_family(hs, f, 48, kinds=[0, 1])


def test_conf_llama_entropy_vocab(hs):
    fam = synth.FAMILIES["c4"]
    check_family(hs, fam, 24, kinds=[2, 0])


@pytest.mark.parametrize("T", [0.05, 1.0, 20.0])
def test_conf_temperatures(hs, T):
    check_family(hs, synth.FAMILIES["c2"], 2000, kinds=[0, 2], T=T)


def test_conf_adversarial_rows(hs):
    C = 64
    rows = []
    rows.append(np.zeros(C))                                    # uniform, tie at 0
    r = np.full(C, -3.0); r[[5, 9, 40]] = 7.0; rows.append(r)     # 3-way tie
    r = np.full(C, -np.inf); r[[3, 4]] = 1.0; rows.append(r)     # masked classes
    r = np.full(C, -np.inf); r[60] = -2.0; rows.append(r)        # one live class
    r = np.zeros(C); r[0] = 1e30; rows.append(r)                 # huge (fp32 only)
    r = np.linspace(-50, 50, C); rows.append(r)                  # ramp
    r = np.zeros(C); r[7] = 88.0; rows.append(r)                 # saturated
    r = np.zeros(C); r[1] = np.nan; rows.append(r)               # NaN -> invalid
    r = np.zeros(C); r[2] = np.inf; rows.append(r)               # +inf -> invalid
    rows.append(np.full(C, -np.inf))                             # all masked -> invalid
    r = np.full(C, 1e-40); r[11] = 2e-40; rows.append(r)         # denormals
    x32 = np.stack(rows).astype(np.float32)
    for dtype in ("fp32", "bf16"):
        bits = x32 if dtype == "fp32" else torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
        x = to_dev_bits(bits, dtype)
        for kind in (0, 1, 2):
            for T in (0.05, 1.0, 20.0):
                r, st = run_conf(hs, x, None, len(rows), 1, C, T, kind, 0)
                ref = oracle.confidence(host_bits(x), len(rows), 1, C, C, T, kind=kind)
                assert st == 1, "invalid rows must set status bit 0"
                assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
                assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"])


def _adversarial_rows(C: int, rng) -> np.ndarray:
    """Hard rows at the width C of a production launch shape: random normal at
    several scales (not the generator's quantised values), exact ties, masked
    classes, huge and subnormal magnitudes, NaN / +inf / all -inf (invalid)."""
    rows = []
    for scale in (0.01, 1.0, 4.0, 30.0):
        for _ in range(3):
            rows.append(rng.normal(0.0, scale, C))
    r = rng.normal(0, 1, C); r[[1, C // 2, C - 1]] = r.max() + 1.0; rows.append(r)   # 3-way tie
    r = rng.normal(0, 1, C); r[C - 1] = r.max() + 0.5; rows.append(r)                # max in the ragged tail
    r = rng.normal(0, 2, C); r[rng.random(C) < 0.5] = -np.inf; rows.append(r)        # half masked
    r = np.full(C, -np.inf); r[C // 3] = -5.0; rows.append(r)                        # one live class
    rows.append(np.zeros(C))                                                         # uniform
    r = np.full(C, 1e-40); r[7] = 3e-40; rows.append(r)                              # subnormal max
    r = rng.normal(0, 1, C); r[5] = 60.0; rows.append(r)                             # saturated
    r = rng.normal(0, 1, C); r[C // 2] = np.nan; rows.append(r)                      # invalid
    r = rng.normal(0, 1, C); r[0] = np.inf; rows.append(r)                           # invalid
    rows.append(np.full(C, -np.inf))                                                 # invalid
    return np.stack(rows).astype(np.float32)


@pytest.mark.parametrize("C,dtype", [(1000, "bf16"), (1000, "fp32"), (32128, "bf16"), (128256, "bf16")])
@pytest.mark.parametrize("T", [0.05, 1.0, 20.0])
def test_conf_production_shapes_random_and_adversarial(hs, C, dtype, T):
    """The production instantiations the bench runs (K1a for C = 1,000: bf16
    NV=8/G=16 and fp32; K1d for the T5 / Llama vocabularies, forced by a
    workspace without the split-row region) on random-normal and adversarial
    rows -- not only on the generator's quantised values -- at three
    temperatures, every confidence kind, against the fp64 oracle."""
    rng = np.random.default_rng(C + int(T * 100))
    x32 = _adversarial_rows(C, rng)
    # repeat so that a K1a launch covers many row groups and warps
    reps = 40 if C <= 4096 else 1
    x32 = np.concatenate([x32] * reps)
    if dtype == "bf16":
        bits = torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    else:
        bits = x32
    n = bits.shape[0]
    x = to_dev_bits(bits, dtype)
    lab = (np.arange(n) * 7919 % C).astype(np.int32)
    lab_d = torch.from_numpy(lab).to(dev())
    ws = torch.zeros(16, dtype=torch.uint8, device=dev())        # no split region: K1a / K1d
    for kind in (0, 1, 2):
        st = torch.zeros(1, dtype=torch.int32, device=dev())
        r = hs.confidence(x, n_classes=C, temperature=T, kind=kind, labels=lab_d, status=st, ws=ws)
        torch.cuda.synchronize()
        ref = oracle.confidence(host_bits(x), n, 1, C, C, T, kind=kind, labels=lab)
        assert int(st.item()) == 1
        assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
        assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"])
        assert np.array_equal(r["correct"].cpu().numpy(), ref["correct"])


def test_conf_row_index_and_dynamic_n(hs):
    fam = synth.FAMILIES["c2"]
    n_all = 5000
    bits = synth.fam_logits_np(fam, 1, np.arange(n_all), "bf16", L=1, C=fam.C)
    x = to_dev_bits(bits, "bf16")
    ri = np.sort(np.random.default_rng(0).choice(n_all, 1234, replace=False))
    r, _ = run_conf(hs, x, fam, len(ri), 1, fam.C, 1.3, 0, 0, row_index=ri)
    ref = oracle.confidence(bits, len(ri), 1, fam.C, fam.C, 1.3, row_index=ri)
    assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
    # device-side count: only the first d_n items are processed
    d_n = torch.tensor([700], dtype=torch.int64, device=dev())
    out = {"conf": torch.full((1234,), -7.0, device=dev())}
    hs.confidence(x, n=1234, n_classes=fam.C, temperature=1.3, d_n=d_n, out=out,
                  row_index=torch.from_numpy(ri).to(dev()))
    g = out["conf"].cpu().numpy()
    assert_conf_close(g[:700], ref["conf"][:700])
    assert np.all(g[700:] == -7.0)


def test_gpu_generator_matches_numpy(hs):
    import workload
    for key in ("c1", "c2", "c3", "c4", "c5"):
        fam = synth.FAMILIES[key]
        L = min(fam.L, 3)
        f = synth.scaled(fam, L=L)
        ids = np.array([0, 1, 5, 77, 1 << 33], np.int64)
        want = synth.fam_logits_np(f, 1, ids, f.dtype, L=L, C=f.C)
        tdt = torch.bfloat16 if f.dtype == "bf16" else torch.float32
        out = torch.empty(len(ids) * L, f.C, dtype=tdt, device=dev())
        workload.gpu_logits(out, f, 1, ids=torch.from_numpy(ids).to(dev()))
        assert np.array_equal(host_bits(out), want)
        lab = torch.empty(len(ids) * L, dtype=torch.int32, device=dev())
        workload.gpu_labels(lab, f, ids=torch.from_numpy(ids).to(dev()))
        assert np.array_equal(lab.cpu().numpy(), synth.labels_np(f.seed, ids, L, f.C).reshape(-1))


# ---------------------------------------------------------------------------
# K3/K4 routing + compaction
# ---------------------------------------------------------------------------
def _route_ref(conf32: np.ndarray, t: float, is_last: bool):
    return oracle.route(conf32.astype(np.float64), float(np.float32(t)), is_last)


@pytest.mark.parametrize("n", [0, 1, 31, 2047, 2048, 2049, 4095, 4096, 4097, 12289, 262144])
def test_route_compact_exact(hs, n):
    rng = np.random.default_rng(n)
    c = rng.uniform(size=n).astype(np.float32)
    if n:
        c[rng.uniform(size=n) < 0.02] = np.nan
        c[rng.uniform(size=n) < 0.05] = np.float32(0.5)         # exact ties with t
    cd = torch.from_numpy(c).to(dev())
    ids = torch.from_numpy(rng.integers(0, 1 << 40, size=n)).to(dev())
    pred = torch.from_numpy(rng.integers(0, 1000, size=3 * n).astype(np.int32)).to(dev())
    payload = torch.from_numpy(rng.integers(0, 255, size=(n, 48), dtype=np.uint8)).to(dev())
    ws = hs.workspace(hs.lib().hs_route_compact_workspace(n), dev())
    for t, last in ((0.5, False), (0.0, False), (1.0, False), (math.inf, False), (0.3, True)):
        o = hs.route_compact(cd, t, is_last=last, ids=ids, pred=pred, pred_len=3, payload=payload,
                             ws=ws)
        torch.cuda.synchronize()
        acc, dfr = _route_ref(c, t, last)
        na, nd = o["counts"].cpu().tolist()
        assert (na, nd) == (len(acc), len(dfr))
        idh = ids.cpu().numpy()
        assert np.array_equal(o["acc_ids"][:na].cpu().numpy(), idh[acc])
        assert np.array_equal(o["def_ids"][:nd].cpu().numpy(), idh[dfr])
        assert np.array_equal(o["def_pos"][:nd].cpu().numpy(), dfr)
        np.testing.assert_array_equal(o["acc_conf"][:na].cpu().numpy(), c[acc])
        assert np.array_equal(o["acc_pred"][:3 * na].cpu().numpy().reshape(-1, 3),
                              pred.cpu().numpy().reshape(-1, 3)[acc])
        if not last:
            assert np.array_equal(o["def_payload"][:nd].cpu().numpy(), payload.cpu().numpy()[dfr])
    # the workspace is reused across calls without a memset (epoch-tagged descriptors)
    epoch = int(ws[:4].view(torch.int32).item())
    assert epoch == (5 if n > 0 else 0)


@pytest.mark.parametrize("n", [1, 7, 8, 9, 2047, 2048, 2049, 6151, 262144, 300001])
@pytest.mark.parametrize("offset", [0, 1])
def test_route_compact_fast_path(hs, n, offset):
    """The plain cascade split (pred_len = 1 or no pred): 8 consecutive items per
    thread, 128-bit loads when aligned (offset 0) and scalar loads otherwise
    (offset 1 shifts every array by one element), staged coalesced stores."""
    rng = np.random.default_rng(1000 + n + offset)
    c = rng.uniform(size=n + offset).astype(np.float32)
    c[rng.uniform(size=n + offset) < 0.02] = np.nan
    c[rng.uniform(size=n + offset) < 0.05] = np.float32(0.5)
    ids_all = torch.from_numpy(rng.integers(0, 1 << 40, size=n + offset)).to(dev())
    pred_all = torch.from_numpy(rng.integers(0, 1000, size=n + offset).astype(np.int32)).to(dev())
    cd = torch.from_numpy(c).to(dev())[offset:]
    ids, pred = ids_all[offset:], pred_all[offset:]
    ch = c[offset:]
    ws = hs.workspace(hs.lib().hs_route_compact_workspace(n), dev())
    for t, last, with_ids, with_pred in ((0.5, False, True, True), (0.0, False, False, True),
                                         (math.inf, False, True, False), (0.25, True, True, True),
                                         (0.9, False, False, False)):
        o = hs.route_compact(cd, t, is_last=last, ids=ids if with_ids else None,
                             pred=pred if with_pred else None, pred_len=1, ws=ws)
        torch.cuda.synchronize()
        acc, dfr = _route_ref(ch, t, last)
        na, nd = o["counts"].cpu().tolist()
        assert (na, nd) == (len(acc), len(dfr)), (t, last)
        idh = ids.cpu().numpy() if with_ids else np.arange(n)
        assert np.array_equal(o["acc_ids"][:na].cpu().numpy(), idh[acc])
        assert np.array_equal(o["def_ids"][:nd].cpu().numpy(), idh[dfr])
        assert np.array_equal(o["def_pos"][:nd].cpu().numpy(), dfr)
        np.testing.assert_array_equal(o["acc_conf"][:na].cpu().numpy(), ch[acc])
        if with_pred:
            assert np.array_equal(o["acc_pred"][:na].cpu().numpy(), pred.cpu().numpy()[acc])


def test_route_device_threshold_and_count(hs):
    rng = np.random.default_rng(5)
    n = 20000
    c = rng.uniform(size=n).astype(np.float32)
    cd = torch.from_numpy(c).to(dev())
    d_n = torch.tensor([15000], dtype=torch.int64, device=dev())
    d_t = torch.tensor([0.625], dtype=torch.float32, device=dev())
    o = hs.route_compact(cd, d_t, n=n, d_n=d_n)
    torch.cuda.synchronize()
    acc, dfr = _route_ref(c[:15000], 0.625, False)
    assert o["counts"].cpu().tolist() == [len(acc), len(dfr)]
    assert np.array_equal(o["acc_ids"][:len(acc)].cpu().numpy(), acc)


# ---------------------------------------------------------------------------
# Whole cascade (K1 -> K3 -> K4 per stage, device-resident counts/thresholds)
# ---------------------------------------------------------------------------
def near_per_stage(conf_by_stage, t, stage_of=None):
    """request r is near-threshold at stage k when it reaches k
    (on the oracle's path) and |c_k(r) - t_k| <= 1e-5 * t_k.  Returns the mask of
    requests near at some stage (removed from both sides' lists at every stage)
    and the count per stage (reported)."""
    n = conf_by_stage.shape[1]
    if stage_of is None:
        stage_of = oracle.cascade(conf_by_stage, np.asarray(t, np.float64))
    near = np.zeros(n, bool)
    counts = []
    for k in range(len(t) - 1):
        nk = np.zeros(n, bool)
        if np.isfinite(t[k]):
            nk = (stage_of >= k) & (np.abs(conf_by_stage[k] - t[k]) <= REL * t[k])
        counts.append(int(nk.sum()))
        near |= nk
    return near, counts


def near_mask(conf_by_stage, t):
    return near_per_stage(conf_by_stage, t)[0]


@pytest.mark.parametrize("key,n", [("c1", 4096), ("c2", 20000), ("c4", 96)])
def test_cascade_vs_oracle(hs, key, n):
    fam = synth.FAMILIES[key]
    K = fam.K
    ids = np.arange(n, dtype=np.int64)
    logits, conf_o = [], []
    for k in range(K):
        bits = synth.fam_logits_np(fam, k, ids, fam.dtype, L=fam.L, C=fam.C)
        logits.append(to_dev_bits(bits, fam.dtype))
        conf_o.append(oracle.confidence(bits, n, fam.L, fam.C, fam.C, fam.temps[k], kind=fam.kind,
                                        reduce=fam.reduce)["conf"])
    conf_o = np.stack(conf_o)
    rng = np.random.default_rng(1)
    t = np.sort(rng.uniform(0.2, 0.9, size=K - 1)).astype(np.float32).tolist() + [0.0]
    P = 64
    payload = torch.from_numpy(rng.integers(0, 255, size=(n, P), dtype=np.uint8)).to(dev())
    casc = hs.Cascade(n, [hs.StageSpec(fam.C, fam.temps[k], fam.L, fam.kind, fam.reduce)
                          for k in range(K)], dev(), payload_row_bytes=P)
    casc.route(logits, t, payload=payload)
    res = casc.results()
    tt = np.array(t, np.float64)
    stage_of = oracle.cascade(conf_o, tt)
    lists = oracle.stage_lists(stage_of, K)
    near, near_counts = near_per_stage(conf_o, tt, stage_of)
    print(f"{key}: near-threshold requests per stage {near_counts} of {n}")
    assert near.sum() <= max(3, n // 1000)
    for k in range(K):
        got = res[k]["ids"].numpy()
        want = lists[k][1]
        assert np.array_equal(got[~near[got]], want[~near[want]])
        if k < K - 1 and not near.any():
            batch_next = lists[k][2]
            nd = res[k]["n_def"]
            pl = casc.outs[k]["next_payload"][:nd * P].cpu().numpy().reshape(nd, P)
            assert np.array_equal(pl, payload.cpu().numpy()[batch_next])


# ---------------------------------------------------------------------------
# K5/K6 calibration
# ---------------------------------------------------------------------------
@pytest.mark.parametrize("graph", [False, True])
def test_router_overlap_first_equals_serial(hs, graph):
    """HS_STEP_OVERLAP_PREVIOUS: routing stage 1's K1 runs next to the
    calibration (no early PDL wait, rows claimed from the step ticket).  The
    cascade must equal the strictly serial one bit for bit, eagerly and when
    replayed from a CUDA graph, over repeated steps (ticket re-arming)."""
    from paper_2505_12566_b200.router import Router
    fam = synth.FAMILIES["c2"]
    n, n_val = 131072, 20000
    stages = [hs.StageSpec(fam.C, fam.temps[k], fam.L, fam.kind, fam.reduce) for k in range(fam.K)]
    route, val = [], []
    for k in range(fam.K):
        x = torch.empty(n, fam.C, dtype=torch.bfloat16, device=dev())
        workload.gpu_logits(x, fam, k, n=n)
        route.append(x)
        v = torch.empty(n_val, fam.C, dtype=torch.bfloat16, device=dev())
        workload.gpu_logits(v, fam, k, n=n_val, id_base=synth.VAL_ID_BASE)
        val.append(v)
    lab = torch.empty(n_val, dtype=torch.int32, device=dev())
    workload.gpu_labels(lab, fam, id_base=synth.VAL_ID_BASE, n=n_val)

    def run(overlap):
        r = Router(stages, n, n_val, dev(), log2_bins=fam.log2_bins)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
        with torch.cuda.stream(s):
            def step():
                r.calibrate(val, lab)
                r.route(route, overlap_first=overlap)
            step()
            if graph:
                s.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    step()
                for _ in range(3):
                    g.replay()
            else:
                for _ in range(3):
                    step()
        torch.cuda.synchronize()
        return r.cal["t"].cpu(), r.cascade.results()

    t0, res0 = run(False)
    t1, res1 = run(True)
    assert torch.equal(t0, t1)
    assert [x["n_acc"] for x in res0] == [x["n_acc"] for x in res1]
    for a, b in zip(res0, res1):
        for key in ("ids", "conf", "pred"):
            assert torch.equal(a[key], b[key]), key


def _gpu_val(hs, fam, n_val):
    K = fam.K
    vids = np.arange(n_val, dtype=np.int64) + synth.VAL_ID_BASE
    lab = synth.labels_np(fam.seed, vids, fam.L, fam.C).reshape(-1)
    lab_d = torch.from_numpy(lab).to(dev())
    vconf = torch.empty(K - 1, n_val, dtype=torch.float32, device=dev())
    vok = torch.empty(K, n_val, dtype=torch.uint8, device=dev())
    oconf = np.empty((K - 1, n_val))
    for k in range(K):
        bits = synth.fam_logits_np(fam, k, vids, fam.dtype, L=fam.L, C=fam.C)
        x = to_dev_bits(bits, fam.dtype)
        r = hs.confidence(x, n=n_val, seq_len=fam.L, temperature=fam.temps[k], kind=fam.kind,
                          reduce=fam.reduce, labels=lab_d)
        vok[k] = r["correct"]
        if k < K - 1:
            vconf[k] = r["conf"]
            oconf[k] = oracle.confidence(bits, n_val, fam.L, fam.C, fam.C, fam.temps[k],
                                         kind=fam.kind, reduce=fam.reduce)["conf"]
    return vconf, vok, oconf


@pytest.mark.parametrize("key,n_val,q", [("c1", 4096, 12), ("c2", 50000, 12), ("c2", 3000, 4),
                                         ("c2", 777, 14), ("c4", 256, 10)])
def test_calibration_bit_exact(hs, key, n_val, q):
    fam = synth.FAMILIES[key]
    vconf, vok, oconf = _gpu_val(hs, fam, n_val)
    g = hs.calibrate_thresholds(vconf, vok, log2_bins=q)
    torch.cuda.synchronize()
    gc, gk = vconf.cpu().numpy(), vok.cpu().numpy()
    # (i) oracle on the GPU's confidences and correct bits: bit-exact, no exceptions
    ref = oracle.calibrate(gc, gk, q)
    assert np.array_equal(g["b"].cpu().numpy(), ref["b"])
    assert np.array_equal(g["reach"].cpu().numpy(), ref["reach"])
    assert np.array_equal(g["handled"].cpu().numpy(), ref["handled"])
    assert int(g["correct_total"].item()) == ref["correct_total"] >= ref["tau"]
    assert np.array_equal(g["t"].cpu().numpy().astype(np.float64), ref["t"])
    # (ii) oracle on its own fp64 confidences: equal unless a sample within 1e-5
    # of a bin edge crossed an edge that decides a minimum
    own = oracle.calibrate(oconf, gk, q)
    check_calibration_ii(own["b"], ref["b"], oconf, gc, q)


def check_calibration_ii(b_own, b_gpu, oconf, gconf, q):
    """SURVEY 8(c) check (ii).  A sample whose bin differs between the oracle's
    and the GPU's confidence ("flip") must lie within 1e-5 (relative) of the bin
    edge it crosses.  The two calibrations must then agree unless a flip
    decides a minimum: at the first round k where they differ, some flip of an
    earlier round j crossed that round's acceptance edge b_j (it changed the
    alive set / the committed answers), or a flip of round k crossed an edge
    between the two choices of b_k (it changed S(b) there).  Returns the flip
    count (reported)."""
    B = 1 << q
    ob = np.where(np.isnan(oconf), -1, np.minimum(B, np.floor(oconf * B))).astype(np.int64)
    gb = np.where(np.isnan(gconf), -1, np.minimum(B, np.floor(gconf.astype(np.float64) * B))).astype(np.int64)
    flip = ob != gb
    edges = np.maximum(ob, gb)[flip]                 # the edge e: bin e-1 on one side, e on the other
    near = np.abs(oconf[flip] * B - edges) <= REL * np.maximum(oconf[flip] * B, 1e-30)
    assert near.all(), "a sample changed bin although it is not within 1e-5 of the edge"
    assert (np.abs(ob - gb)[flip] == 1).all()
    b_own, b_gpu = np.asarray(b_own), np.asarray(b_gpu)
    if not np.array_equal(b_own, b_gpu):
        k = int(np.flatnonzero(b_own != b_gpu)[0])
        rows = np.nonzero(flip)[0]
        e_by_round = [set(np.maximum(ob, gb)[j][flip[j]].tolist()) for j in range(flip.shape[0])]
        lo, hi = min(b_own[k], b_gpu[k]), max(b_own[k], b_gpu[k])
        deciding = any(int(b_gpu[j]) in e_by_round[j] for j in range(k)) or \
            any(lo <= e <= hi for e in e_by_round[k])
        assert deciding, f"b differs at round {k} without a deciding near-edge sample ({len(rows)} flips)"
    print(f"calibration (ii): {int(flip.sum())} near-edge samples changed bin; b equal: "
          f"{bool(np.array_equal(b_own, b_gpu))}")
    return int(flip.sum())


def test_calibration_blocks_equal_full_call(hs):
    fam = synth.FAMILIES["c2"]
    vconf, vok, _ = _gpu_val(hs, fam, 6000)
    q, K = 11, fam.K
    full = hs.calibrate_thresholds(vconf, vok, log2_bins=q, target=4000)
    ws = hs.calibrate_workspace(K, q, dev())
    out = hs._calib_out(K, dev(), None)
    hs.calibrate_begin(K, q, 4000, ws)
    for k in range(K - 1):
        # two "ranks": each adds its shard's histogram (sum == one big histogram)
        hs.calibrate_histogram(vconf[:, :2500].contiguous(), vok[:, :2500].contiguous(), k,
                               out["b"], log2_bins=q, ws=ws)
        hs.calibrate_histogram(vconf[:, 2500:].contiguous(), vok[:, 2500:].contiguous(), k,
                               out["b"], log2_bins=q, ws=ws)
        hs.calibrate_select(K, k, out, log2_bins=q, ws=ws)
    torch.cuda.synchronize()
    for key in ("b", "t", "reach", "handled", "correct_total"):
        assert torch.equal(full[key], out[key]), key


def test_calibration_degenerate(hs):
    # c = 1.0 exactly is reachable: only defer-all (b = B+1, t = +inf) rejects it (G11)
    conf = torch.tensor([[1.0, 1.0, 0.5]], device=dev())
    ok = torch.tensor([[0, 0, 1], [1, 1, 1]], dtype=torch.uint8, device=dev())
    g = hs.calibrate_thresholds(conf, ok, log2_bins=3)
    assert g["b"].item() == 9 and math.isinf(g["t"][0].item()) and g["correct_total"].item() == 3
    # NaN confidences are never accepted
    conf = torch.tensor([[float("nan"), 0.9]], device=dev())
    ok = torch.tensor([[1, 1], [0, 1]], dtype=torch.uint8, device=dev())
    g = hs.calibrate_thresholds(conf, ok, log2_bins=4)
    ref = oracle.calibrate(conf.cpu().numpy(), ok.cpu().numpy(), 4)
    assert g["b"].cpu().tolist() == ref["b"].tolist() and g["handled"].cpu().tolist() == ref["handled"].tolist()


# ---------------------------------------------------------------------------
# Full BASELINE sizes, in the launch configuration bench.py times
# ---------------------------------------------------------------------------
def test_full_size_c2_sampled(hs):
    import workload
    fam = synth.FAMILIES["c2"]
    n = fam.n
    x = torch.empty(n, fam.C, dtype=torch.bfloat16, device=dev())
    workload.gpu_logits(x, fam, 0, id_base=0, n=n)
    r = hs.confidence(x, temperature=fam.temps[0])
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(2).choice(n, 3000, replace=False))
    sample = host_bits(x[torch.from_numpy(rows).to(dev())])
    ref = oracle.confidence(sample, len(rows), 1, fam.C, fam.C, fam.temps[0])
    assert_conf_close(r["conf"].cpu().numpy()[rows], ref["conf"])
    assert np.array_equal(r["argmax"].cpu().numpy()[rows], ref["argmax"])
    # full-size compaction on these confidences is exact integer work: compare all of it
    c = r["conf"].cpu().numpy()
    o = hs.route_compact(r["conf"], 0.7)
    torch.cuda.synchronize()
    acc, dfr = _route_ref(c, 0.7, False)
    assert o["counts"].cpu().tolist() == [len(acc), len(dfr)]
    assert np.array_equal(o["def_ids"][:len(dfr)].cpu().numpy(), dfr)


def test_full_size_c4_sampled(hs):
    import workload
    fam = synth.FAMILIES["c4"]
    n = fam.n
    x = torch.empty(n, fam.C, dtype=torch.bfloat16, device=dev())
    workload.gpu_logits(x, fam, 0, id_base=0, n=n)
    r = hs.confidence(x, temperature=fam.temps[0], kind="entropy")
    torch.cuda.synchronize()
    rows = np.sort(np.random.default_rng(3).choice(n, 64, replace=False))
    sample = host_bits(x[torch.from_numpy(rows).to(dev())])
    ref = oracle.confidence(sample, len(rows), 1, fam.C, fam.C, fam.temps[0], kind=oracle.ENTROPY)
    assert_conf_close(r["conf"].cpu().numpy()[rows], ref["conf"])
    assert np.array_equal(r["argmax"].cpu().numpy()[rows], ref["argmax"])
    del x


def test_c3_sequences_sampled_launch_config(hs):
    """T5: 64 tokens x 32,128 vocab per sequence, MIN/MEAN; sampled sequences of the full id range."""
    import workload
    fam = synth.FAMILIES["c3"]
    ids = np.sort(np.random.default_rng(4).choice(fam.n, 24, replace=False)).astype(np.int64)
    x = torch.empty(len(ids) * fam.L, fam.C, dtype=torch.bfloat16, device=dev())
    workload.gpu_logits(x, fam, 2, ids=torch.from_numpy(ids).to(dev()))
    lab = torch.empty(len(ids) * fam.L, dtype=torch.int32, device=dev())
    workload.gpu_labels(lab, fam, ids=torch.from_numpy(ids).to(dev()))
    for reduce in ("min", "mean"):
        r = hs.confidence(x, n=len(ids), seq_len=fam.L, temperature=1.0, reduce=reduce, labels=lab)
        torch.cuda.synchronize()
        ref = oracle.confidence(host_bits(x), len(ids), fam.L, fam.C, fam.C, 1.0,
                                reduce=oracle.SEQ_MIN if reduce == "min" else oracle.SEQ_MEAN,
                                labels=lab.cpu().numpy())
        assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
        assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"])
        assert np.array_equal(r["correct"].cpu().numpy(), ref["correct"])


def test_calibration_modes_agree(hs, monkeypatch):
    """One cluster launch (DSMEM histogram merge; default for small sets), one
    cooperative grid launch, and per-round histogram/select launches give
    identical thresholds and counts."""
    fam = synth.FAMILIES["c2"]
    vconf, vok, _ = _gpu_val(hs, fam, 20000)
    for q in (3, 12, 14):
        res = {}
        for mode in ("cluster", "fused", "fused_streaming", "split"):
            monkeypatch.setenv("HS_CALIB_MODE", mode.split("_")[0])
            if mode == "fused_streaming":          # the non-resident cooperative kernel
                monkeypatch.setenv("HS_CALIB_NORESIDENT", "1")
            res[mode] = hs.calibrate_thresholds(vconf, vok, log2_bins=q)
            monkeypatch.delenv("HS_CALIB_NORESIDENT", raising=False)
        monkeypatch.delenv("HS_CALIB_MODE")
        torch.cuda.synchronize()
        ref = oracle.calibrate(vconf.cpu().numpy(), vok.cpu().numpy(), q)
        for mode, r in res.items():
            assert np.array_equal(r["b"].cpu().numpy(), ref["b"]), (q, mode)
            for key in ("b", "t", "reach", "handled", "correct_total"):
                assert torch.equal(r[key], res["split"][key]), (q, mode, key)


@pytest.mark.parametrize("K,N,q", [(2, 1, 12), (3, 4095, 8), (7, 300001, 12), (16, 70000, 10),
                                   (4, 100000, 14), (3, 20000, 13), (6, 200000, 1), (5, 50000, 11),
                                   (5, 1 << 22, 12)])
def test_calibration_resident_vs_streaming(hs, monkeypatch, K, N, q):
    """The resident cooperative kernel (samples in shared memory, three rotating
    histograms, redundant per-CTA select) == the streaming one == the oracle.
    The last case does not fit shared memory and exercises the fallback."""
    g = torch.Generator().manual_seed(K * 1000 + q)
    conf = torch.rand(K - 1, N, generator=g)
    conf[:, ::97] = float("nan")
    conf[:, 1::89] = 1.0
    ok = (torch.rand(K, N, generator=g) < 0.75).to(torch.uint8)
    d_conf, d_ok = conf.to(dev()), ok.to(dev())
    res = {}
    for mode in ("resident", "streaming"):
        if mode == "streaming":
            monkeypatch.setenv("HS_CALIB_NORESIDENT", "1")
        res[mode] = hs.calibrate_thresholds(d_conf, d_ok, log2_bins=q)
        monkeypatch.delenv("HS_CALIB_NORESIDENT", raising=False)
    torch.cuda.synchronize()
    for key in ("b", "t", "reach", "handled", "correct_total"):
        assert torch.equal(res["resident"][key], res["streaming"][key]), key
    if N <= 300001:
        ref = oracle.calibrate(conf.numpy(), ok.numpy(), q)
        assert np.array_equal(res["resident"]["b"].cpu().numpy(), ref["b"])
        assert int(res["resident"]["correct_total"]) == ref["correct_total"]


@pytest.mark.parametrize("key,n_val", [("c2", 3001), ("c1", 513), ("c4", 24)])
def test_confidence_batched_equals_per_stage(hs, key, n_val):
    """hs_confidence_batched (all stages in one launch) == K separate hs_confidence calls == oracle."""
    fam = synth.FAMILIES[key]
    vids = np.arange(n_val, dtype=np.int64) + synth.VAL_ID_BASE
    lab = synth.labels_np(fam.seed, vids, fam.L, fam.C).reshape(-1)
    lab_d = torch.from_numpy(lab).to(dev())
    bits = [synth.fam_logits_np(fam, k, vids, fam.dtype, L=fam.L, C=fam.C) for k in range(fam.K)]
    xs = [to_dev_bits(b, fam.dtype) for b in bits]
    got = hs.confidence_batched(xs, fam.temps, n=n_val, seq_len=fam.L, kind=fam.kind,
                                reduce=fam.reduce, labels=lab_d)
    torch.cuda.synchronize()
    for k in range(fam.K):
        one = hs.confidence(xs[k], n=n_val, seq_len=fam.L, temperature=fam.temps[k], kind=fam.kind,
                            reduce=fam.reduce, labels=lab_d)
        torch.cuda.synchronize()
        sl = slice(k * n_val, (k + 1) * n_val)
        # one launch per stage may take the split-row path for a few long rows
        # (another reduction order): equal within the K1 tolerance, not bitwise
        g1, o1 = got["conf"][sl].cpu().numpy(), one["conf"].cpu().numpy()
        assert np.array_equal(np.isnan(g1), np.isnan(o1))
        assert np.allclose(g1, o1, rtol=REL, atol=0, equal_nan=True)
        assert torch.equal(got["correct"][sl], one["correct"])
        assert torch.equal(got["argmax"][k * n_val * fam.L:(k + 1) * n_val * fam.L], one["argmax"])
        ref = oracle.confidence(bits[k], n_val, fam.L, fam.C, fam.C, fam.temps[k], kind=fam.kind,
                                reduce=fam.reduce, labels=lab)
        assert_conf_close(got["conf"][sl].cpu().numpy(), ref["conf"])
        assert np.array_equal(got["correct"][sl].cpu().numpy(), ref["correct"])


@pytest.mark.parametrize("passes", [1, 3])
@pytest.mark.parametrize("q", [4, 12])
def test_calibration_refinement_bit_exact(hs, passes, q):
    """GPU refinement passes == oracle refinement (same thresholds, counts, correct total)."""
    fam = synth.FAMILIES["c2"]
    vconf, vok, _ = _gpu_val(hs, fam, 20000)
    g = hs.calibrate_thresholds(vconf, vok, log2_bins=q, refine_passes=passes)
    greedy = hs.calibrate_thresholds(vconf, vok, log2_bins=q)
    torch.cuda.synchronize()
    ref = oracle.calibrate(vconf.cpu().numpy(), vok.cpu().numpy(), q, refine_passes=passes)
    assert np.array_equal(g["b"].cpu().numpy(), ref["b"])
    assert np.array_equal(g["reach"].cpu().numpy(), ref["reach"])
    assert np.array_equal(g["handled"].cpu().numpy(), ref["handled"])
    assert int(g["correct_total"].item()) == ref["correct_total"] >= ref["tau"]
    assert np.array_equal(g["t"].cpu().numpy().astype(np.float64), ref["t"])
    assert np.all(g["b"].cpu().numpy() <= greedy["b"].cpu().numpy())     # never raises b_k


def test_calibration_refinement_small_random(hs):
    """Random small validation sets (K <= 5, N <= 300) incl. NaN confidences."""
    rng = np.random.default_rng(11)
    for _ in range(30):
        K = int(rng.integers(3, 6))
        N = int(rng.integers(1, 300))
        q = int(rng.integers(1, 6))
        d = rng.uniform(size=N)
        ok = np.stack([(d + 0.3 * rng.normal(size=N) < 0.5 + 0.1 * k) for k in range(K)]).astype(np.uint8)
        conf = np.clip(np.where(ok[:-1] == 1, rng.beta(5, 2, (K - 1, N)), rng.beta(2, 3, (K - 1, N))), 0, 1)
        conf[rng.uniform(size=conf.shape) < 0.03] = np.nan
        c = torch.from_numpy(conf.astype(np.float32)).to(dev())
        o = torch.from_numpy(ok).to(dev())
        for passes in (0, 2):
            g = hs.calibrate_thresholds(c, o, log2_bins=q, refine_passes=passes)
            torch.cuda.synchronize()
            ref = oracle.calibrate(conf.astype(np.float32).astype(np.float64), ok, q, refine_passes=passes)
            assert np.array_equal(g["b"].cpu().numpy(), ref["b"]), (K, N, q, passes)
            assert np.array_equal(g["handled"].cpu().numpy(), ref["handled"])
            assert int(g["correct_total"].item()) == ref["correct_total"]


# ---------------------------------------------------------------------------
# NEXT-1 skip connections
# ---------------------------------------------------------------------------
def test_skip_edges_match_oracle(hs):
    # the C-ABI takes the fp32 threshold the router compares against (D3)
    for t in (0.0, 0.25, 0.7, 0.999, 1.0):
        t32 = float(np.float32(t))
        for s_ in range(1, 8):
            for mode in (0, 1):
                assert np.array_equal(np.array(hs.skip_edges(t32, s_, mode), np.float32),
                                      oracle.skip_edges(t32, s_, mode)), (t, s_, mode)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("key,n", [("c2", 20000), ("c1", 4096)])
def test_skip_cascade_vs_oracle(hs, mode, key, n):
    fam = synth.FAMILIES[key]
    K = fam.K
    ids = np.arange(n, dtype=np.int64)
    logits, conf_o = [], []
    for k in range(K):
        bits = synth.fam_logits_np(fam, k, ids, fam.dtype, L=fam.L, C=fam.C)
        logits.append(to_dev_bits(bits, fam.dtype))
        conf_o.append(oracle.confidence(bits, n, fam.L, fam.C, fam.C, fam.temps[k], kind=fam.kind,
                                        reduce=fam.reduce)["conf"])
    conf_o = np.stack(conf_o)
    t = [0.9, 0.8, 0.7, 0.6, 0.0][-K:] if K > 2 else [0.8, 0.0]
    t = np.array(t, np.float32).astype(np.float64)
    sc = hs.SkipCascade(n, [hs.StageSpec(fam.C, fam.temps[k], fam.L, fam.kind, fam.reduce)
                            for k in range(K)], dev(), mode=mode)
    sc.route(logits, t.tolist())
    res = sc.results()
    stage_of, visits = oracle.cascade_skip(conf_o, t, mode)
    lists = oracle.skip_stage_lists(stage_of, visits, K)
    # requests near a threshold or a band edge may legitimately differ: exclude them
    near = np.zeros(n, bool)
    for k in range(K - 1):
        near |= np.abs(conf_o[k] - t[k]) <= REL * t[k]
        for e in oracle.skip_edges(t[k], K - 1 - k, mode):
            near |= np.abs(conf_o[k] - e) <= REL * max(float(e), 1e-30)
    for k in range(K):
        gb, ga = res[k]["batch"].numpy(), res[k]["ids"].numpy()
        wb, wa = lists[k]
        assert np.array_equal(gb[~near[gb]], wb[~near[wb]]), k
        assert np.array_equal(ga[~near[ga]], wa[~near[wa]]), k
    d = sc.dest.cpu().numpy() - K
    assert np.array_equal(d[~near], stage_of[~near])
    if mode == 0 and K > 2:
        assert (visits & 2 == 0).sum() > 0          # some requests really skipped model 2


# ---------------------------------------------------------------------------
# NEXT-2: Top-K restricted confidence (reading G4): K1c vs oracle
# ---------------------------------------------------------------------------
def _topk_rows(rng, rows, C, mode):
    if mode == "normal":
        return rng.normal(scale=3.0, size=(rows, C)).astype(np.float32)
    if mode == "ties":         # quantised codes: many equal values around the K-th place
        return (rng.integers(-40, 40, size=(rows, C)) * 0.0625).astype(np.float32)
    if mode == "ascending":    # worst case for the first-chunk seed
        return np.tile(np.linspace(-20, 20, C, dtype=np.float32), (rows, 1))
    if mode == "descending":
        return np.tile(np.linspace(20, -20, C, dtype=np.float32), (rows, 1))
    if mode == "masked":       # few finite classes: fewer than K finite values per row
        x = np.full((rows, C), -np.inf, np.float32)
        for i in range(rows):
            j = rng.choice(C, size=min(C, 1 + i % 5), replace=False)
            x[i, j] = rng.normal(size=j.size)
        return x
    if mode == "tiny":         # zeros and subnormals around the maximum
        x = np.zeros((rows, C), np.float32)
        x[:, ::3] = np.float32(1e-40)
        x[:, 1::7] = np.float32(-1e-41)
        return x
    raise ValueError(mode)


def _bf16_bits(x32: np.ndarray) -> np.ndarray:
    return (torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16))


@pytest.mark.parametrize("C", [2, 7, 129, 1000, 4099, 32128])
@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
def test_topk_confidence_vs_oracle(hs, C, dtype):
    rng = np.random.default_rng(C + (1 if dtype == "bf16" else 0))
    rows = 24 if C > 10000 else 96
    for mode in ("normal", "ties", "ascending", "descending", "masked", "tiny"):
        x32 = _topk_rows(rng, rows, C, mode)
        bits = _bf16_bits(x32) if dtype == "bf16" else x32
        x = to_dev_bits(bits, dtype, (C + 7) // 8 * 8)
        lab = rng.integers(0, C, size=rows).astype(np.int32)
        for K in (1, 2, 10, 32):
            for T, kind in ((1.0, 0), (0.05, 1), (20.0, 2)):
                r = hs.confidence(x, n=rows, n_classes=C, temperature=T, kind=kind, top_k=K,
                                  labels=torch.from_numpy(lab).to(dev()))
                torch.cuda.synchronize()
                ref = oracle.confidence(host_bits(x), rows, 1, C, x.stride(0), T, kind=kind,
                                        top_k=K, labels=lab)
                assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
                assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"]), (mode, K)
                assert np.array_equal(r["correct"].cpu().numpy(), ref["correct"]), (mode, K)


def test_topk_invalid_rows_and_full_fallback(hs):
    C = 300
    x32 = np.random.default_rng(3).normal(size=(6, C)).astype(np.float32)
    x32[0, 5] = np.nan
    x32[1, 7] = np.inf
    x32[2, :] = -np.inf
    x = to_dev_bits(x32, "fp32")
    st = torch.zeros(1, dtype=torch.int32, device=dev())
    r = hs.confidence(x, n=6, n_classes=C, top_k=8, status=st)
    torch.cuda.synchronize()
    c = r["conf"].cpu().numpy()
    assert np.isnan(c[:3]).all() and not np.isnan(c[3:]).any() and int(st.item()) & 1
    assert (r["argmax"].cpu().numpy()[:3] == -1).all()
    # top_k >= C is the full softmax
    full = hs.confidence(x, n=6, n_classes=C)["conf"].cpu().numpy()
    big = hs.confidence(x, n=6, n_classes=C, top_k=32)["conf"].cpu().numpy()
    x2 = to_dev_bits(x32[:, :20].copy(), "fp32")
    a = hs.confidence(x2, n=6, n_classes=20, top_k=32)["conf"].cpu().numpy()
    b = hs.confidence(x2, n=6, n_classes=20)["conf"].cpu().numpy()
    torch.cuda.synchronize()
    assert np.array_equal(a, b, equal_nan=True)
    assert not np.array_equal(big[3:], full[3:])        # 32 < 300: restricted
    with pytest.raises(Exception):
        hs.confidence(x, n=6, n_classes=C, top_k=33)


def test_topk_generation_sequences_vs_oracle(hs):
    """C3-like: T5 vocabulary, 64-token sequences, MIN over tokens of the top-K
    restricted confidence, gathered rows."""
    fam = synth.FAMILIES["c3"]
    n = 6
    ids = np.array([5, 0, 17, 3, 9, 11], np.int64)
    bits = synth.fam_logits_np(fam, 1, np.arange(18, dtype=np.int64))
    x = to_dev_bits(bits, fam.dtype)
    lab = synth.labels_np(fam.seed, np.arange(18, dtype=np.int64), fam.L, fam.C).reshape(-1)
    for K, reduce in ((10, oracle.SEQ_MIN), (4, oracle.SEQ_MEAN)):
        r = hs.confidence(x, n=n, seq_len=fam.L, n_classes=fam.C, temperature=fam.temps[1],
                          kind=1, reduce=reduce, top_k=K, row_index=torch.from_numpy(ids).to(dev()),
                          labels=torch.from_numpy(lab).to(dev()))
        torch.cuda.synchronize()
        ref = oracle.confidence(bits, n, fam.L, fam.C, fam.C, fam.temps[1], kind=1, reduce=reduce,
                                row_index=ids, labels=lab, top_k=K)
        assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
        assert np.array_equal(r["argmax"].cpu().numpy(), ref["argmax"])
        assert np.array_equal(r["correct"].cpu().numpy(), ref["correct"])


def test_topk_cascade_step_vs_oracle(hs):
    """A 3-stage cascade whose stages use top-K confidence (StageSpec.top_k)."""
    rng = np.random.default_rng(21)
    n, C, K = 3000, 4096, 8
    xs, conf_o = [], []
    for k in range(3):
        x32 = rng.normal(scale=2.0 + k, size=(n, C)).astype(np.float32)
        bits = _bf16_bits(x32)
        xs.append(to_dev_bits(bits, "bf16"))
        conf_o.append(oracle.confidence(bits, n, 1, C, C, 1.0, kind=0, top_k=K)["conf"])
    conf_o = np.stack(conf_o)
    t = [0.55, 0.45, 0.0]
    casc = hs.Cascade(n, [hs.StageSpec(C, 1.0, 1, 0, 0, top_k=K) for _ in range(3)], dev())
    casc.route(xs, t)
    res = casc.results()
    tt = np.array(np.float32(t), np.float64)
    stage_of = oracle.cascade(conf_o, tt)
    lists = oracle.stage_lists(stage_of, 3)
    near = near_mask(conf_o, tt)
    for k in range(3):
        got, want = res[k]["ids"].numpy(), lists[k][1]
        assert np.array_equal(got[~near[got]], want[~near[want]])


@pytest.mark.parametrize("C,dtype,kind", [(1000, "bf16", 0), (1000, "fp32", 1), (32128, "bf16", 0),
                                          (128256, "bf16", 2), (17, "fp32", 0)])
def test_conf_entropy_alongside(hs, C, dtype, kind):
    """hs_confidence_ex: the entropy confidence exp(-H) written next to the
    requested kind in the same pass (north_star "max-probability (and
    entropy) confidence"), both within 1e-5 of the oracle, on random and
    adversarial rows (invalid rows: NaN in both)."""
    rng = np.random.default_rng(C + kind)
    x32 = _adversarial_rows(C, rng)
    bits = x32 if dtype == "fp32" else \
        torch.from_numpy(x32).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    n = bits.shape[0]
    ve = 8 if dtype == "bf16" else 4
    x = to_dev_bits(bits, dtype, C + (-C) % ve)       # rows padded to 16 bytes
    for ws in (None, torch.zeros(16, dtype=torch.uint8, device=dev())):
        r = hs.confidence(x, n_classes=C, temperature=0.7, kind=kind, want_entropy=True, ws=ws)
        torch.cuda.synchronize()
        st = x.shape[1]
        ref = oracle.confidence(host_bits(x), n, 1, C, st, 0.7, kind=kind)
        ent = oracle.confidence(host_bits(x), n, 1, C, st, 0.7, kind=2)
        assert_conf_close(r["conf"].cpu().numpy(), ref["conf"])
        assert_conf_close(r["conf_entropy"].cpu().numpy(), ent["conf"])
    with pytest.raises(hs.HsError):
        hs.confidence(x, n=n // 2, seq_len=2, n_classes=C, reduce=1, want_entropy=True)


@pytest.mark.parametrize("graph", [False, True])
def test_split_compaction_equals_step(hs, graph):
    """hs_cascade_confidence (+ deferred count) / hs_cascade_compact on a side
    stream -- the compaction off the critical path -- gives the cascade of
    hs_cascade_step bit for bit (dense stage batches, stage 1 overlapping the
    calibration), eagerly and replayed from a CUDA graph, over repeated steps."""
    import bench
    fam = synth.scaled(synth.FAMILIES["c2"], n=65536, n_val=20000)
    route, val, labels, payload = bench.build_inputs(fam, 0, dev())
    base = bench.make_router(fam, dev(), None)
    dense, _ = bench.dense_stage_logits(fam, base, route, val, labels, payload, 0, dev())

    def run(split):
        r = bench.make_router(fam, dev(), None)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
        with torch.cuda.stream(s):
            def step():
                r.calibrate(val, labels)
                r.route(dense, overlap_first=True, by_id=False, split=split)
            step()
            if graph:
                s.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    step()
                for _ in range(3):
                    g.replay()
            else:
                for _ in range(3):
                    step()
        torch.cuda.synchronize()
        return r.cascade.counts.cpu(), r.cascade.results()

    c0, res0 = run(False)
    c1, res1 = run(True)
    assert torch.equal(c0, c1)
    for a, b in zip(res0, res1):
        for key in ("ids", "conf", "pred"):
            assert torch.equal(a[key], b[key]), key
