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
