"""Parity at BASELINE.json's full per-GPU sizes, in the launch configuration
bench.py times: the bench's Router (batched validation confidence, resident
calibration kernel, K-stage cascade with stage 1 overlapping the calibration)
captured in ONE CUDA graph and replayed.  Checked against the oracle on sampled
outputs (confidences of sampled rows, the answering model of sampled requests
under the G18 near-threshold protocol) and through properties that hold at any
size (calibration bit-exact from the GPU's own validation confidences, the
per-stage lists partition the requests, stay sorted and respect the
thresholds)."""
import numpy as np
import pytest
import torch

import oracle

pytestmark = pytest.mark.gpu
REL = 1e-5


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def host_bits(x):
    return x.view(torch.int16).cpu().numpy().view(np.uint16)


@pytest.mark.parametrize("config", ["c2", "c5"])
def test_bench_step_full_size(hs, config):
    import bench
    dev = torch.device("cuda:0")
    fam = bench.family(config)
    route, val, labels, payload = bench.build_inputs(fam, 0, dev)
    router = bench.make_router(fam, dev, None)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far

    def step():
        router.calibrate(val, labels)
        router.route(route, payload=payload, overlap_first=True)

    with torch.cuda.stream(stream):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    K, n, nv = fam.K, fam.n, fam.n_val
    assert int(router.status.item()) == 0
    # 1. validation confidences: sampled rows vs the oracle
    vconf = router.vconf_all.view(K, nv).cpu().numpy()
    vok = router.vok.view(K, nv).cpu().numpy()
    lab = labels.cpu().numpy()
    rng = np.random.default_rng(21)
    for k in range(K):
        rows = np.sort(rng.choice(nv, 800, replace=False))
        ref = oracle.confidence(host_bits(val[k][torch.from_numpy(rows).to(dev)]), len(rows), 1, fam.C,
                                fam.C, fam.temps[k], labels=lab[rows])
        err = np.abs(vconf[k][rows] - ref["conf"]) / ref["conf"]
        assert err.max() <= REL
        assert np.array_equal(vok[k][rows], ref["correct"])
    # 2. calibration: bit-exact from the GPU's own confidences / correct bits (D5)
    cal = oracle.calibrate(vconf[: K - 1], vok, fam.log2_bins)
    assert router.cal["b"].cpu().numpy().tolist() == cal["b"].tolist()
    t = router.cal["t"].cpu().numpy().astype(np.float64)
    assert router.cal["correct_total"].item() == cal["correct_total"] >= cal["tau"]
    # 3. routing: the per-stage accepted lists partition 0..n-1, sorted, thresholds respected
    res = router.cascade.results()
    stage_of = np.full(n, -1, np.int64)
    for k, r in enumerate(res):
        ids = r["ids"].numpy()
        assert (np.diff(ids) > 0).all()
        assert (stage_of[ids] == -1).all()
        stage_of[ids] = k
        if k < K - 1:
            assert (r["conf"].numpy().astype(np.float64) >= t[k]).all()
        if k > 0:
            assert r["n_acc"] + r["n_def"] == res[k - 1]["n_def"]
    assert (stage_of >= 0).all()
    # 4. sampled requests: the answering model equals the oracle's cascade on the
    #    oracle's own confidences (near-threshold requests excluded, G18)
    req = np.sort(rng.choice(n, 3000, replace=False))
    conf_o = np.stack([oracle.confidence(host_bits(route[k][torch.from_numpy(req).to(dev)]), len(req), 1,
                                         fam.C, fam.C, fam.temps[k])["conf"] for k in range(K)])
    near = np.zeros(len(req), bool)
    for k in range(K - 1):
        if np.isfinite(t[k]):
            near |= np.abs(conf_o[k] - t[k]) <= REL * t[k]
    st_o = oracle.cascade(conf_o, t)
    assert np.array_equal(st_o[~near], stage_of[req][~near])
    assert near.sum() <= 5


@pytest.mark.parametrize("config,split", [("c2", True), ("c2", False), ("c4", True)])
def test_bench_dense_step_full_size_every_request(hs, config, split):
    """The TIMED configuration of bench.py (--layout dense, the default): stage
    k's logits are the dense batch of the requests that reach model k; the
    step (batched validation confidence, resident calibration, stage 1
    overlapping it, K stages with device-resident counts) is captured in one
    CUDA graph and replayed.  Every request of every stage batch is checked:
    the oracle's confidence of each dense row decides accept / defer at t_k,
    and the GPU's accepted and deferred lists must equal the oracle's split of
    the same batch, with the near-threshold requests (G18) removed and counted;
    accepted confidences within 1e-5 and predictions bit-exact."""
    import bench
    dev = torch.device("cuda:0")
    fam = bench.family(config)
    route, val, labels, payload = bench.build_inputs(fam, 0, dev)
    router = bench.make_router(fam, dev, None)
    route, _ = bench.dense_stage_logits(fam, router, route, val, labels, payload, 0, dev)
    stream = torch.cuda.Stream(device=dev)
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far

    def step():
        router.calibrate(val, labels)
        router.route(route, payload=payload, overlap_first=True, by_id=False, split=split)

    with torch.cuda.stream(stream):
        step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    K, n = fam.K, fam.n
    assert int(router.status.item()) == 0
    vconf = router.vconf_all.view(K, fam.n_val).cpu().numpy()
    vok = router.vok.view(K, fam.n_val).cpu().numpy()
    cal = oracle.calibrate(vconf[: K - 1], vok, fam.log2_bins)
    assert router.cal["b"].cpu().numpy().tolist() == cal["b"].tolist()
    t = router.cal["t"].cpu().numpy().astype(np.float64)
    counts = router.cascade.counts.cpu().numpy()
    batch_ids = np.arange(n, dtype=np.int64)
    near_counts = []
    for k in range(K):
        nb = len(batch_ids)
        if k:
            assert nb == counts[k - 1][1]
        bits = host_bits(route[k][:nb]) if nb else np.zeros((0, fam.C), np.uint16)
        ref = oracle.confidence(bits, nb, 1, fam.C, fam.C, fam.temps[k], kind=fam.kind)
        last = k == K - 1
        acc_o = np.ones(nb, bool) if last else ref["conf"] >= t[k]
        near = np.zeros(nb, bool) if last else np.abs(ref["conf"] - t[k]) <= REL * t[k]
        near_counts.append(int(near.sum()))
        o = router.cascade.outs[k]
        na, nd = int(counts[k][0]), int(counts[k][1])
        assert na + nd == nb
        acc_ids = o["acc_ids"][:na].cpu().numpy()
        nxt = o["next_ids"][:nd].cpu().numpy() if not last else np.zeros(0, np.int64)
        near_ids = set(batch_ids[near].tolist())
        keep_a = np.array([i not in near_ids for i in acc_ids], bool)
        keep_d = np.array([i not in near_ids for i in nxt], bool)
        assert np.array_equal(acc_ids[keep_a], batch_ids[acc_o & ~near]), k
        assert np.array_equal(nxt[keep_d], batch_ids[~acc_o & ~near]), k
        # accepted confidences and predictions, matched by position in the batch
        pos = np.searchsorted(batch_ids, acc_ids)
        ac = o["acc_conf"][:na].cpu().numpy().astype(np.float64)
        assert (np.abs(ac - ref["conf"][pos]) <= REL * ref["conf"][pos]).all()
        assert np.array_equal(o["acc_pred"][:na].cpu().numpy(), ref["argmax"][pos])
        batch_ids = nxt
    print(f"{config}: near-threshold requests per stage {near_counts}")
    assert sum(near_counts) <= max(5, n // 10000)
