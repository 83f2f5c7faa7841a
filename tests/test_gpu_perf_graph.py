"""GPU parity of NEXT-4, the threshold performance graph (Alg. 1):
hs_threshold_replay + hs_perf_graph vs the oracle (oracle.replay /
oracle.perf_graph).  Every output is an exact integer (correct counts, reach,
energy with integer weights) or an index chosen by exact comparisons, so the
bar is bit-exact; the calibration inputs are the GPU's own fp32 confidences,
so both sides bin the same values (D5 G10)."""
import json
import os

import numpy as np
import pytest
import torch

import oracle
from workload import synth

pytestmark = pytest.mark.gpu
GOLD = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden")


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def dev():
    return torch.device("cuda:0")


def gpu_graph(hs, conf, ok, q, w, bvecs=None, tau=-1, floor=-1, reach=True):
    c = torch.from_numpy(np.ascontiguousarray(conf, np.float32)).to(dev())
    o = torch.from_numpy(np.ascontiguousarray(ok, np.uint8)).to(dev())
    bv = None if bvecs is None else torch.from_numpy(np.ascontiguousarray(bvecs, np.int32)).to(dev())
    r = hs.threshold_replay(c, o, w, log2_bins=q, bvecs=bv, want_reach=reach)
    status = torch.zeros(1, dtype=torch.int32, device=dev())
    g = hs.perf_graph(r["correct"], r["energy"], ok.shape[1], tau=tau, floor=floor,
                      model_correct=r["model_correct"], K=ok.shape[0], status=status)
    torch.cuda.synchronize()
    out = {k: v.cpu().numpy() for k, v in r.items()}
    n = int(g["front_n"].item())
    out.update(front_c=g["front_c"][:n].cpu().numpy(), front_e=g["front_e"][:n].cpu().numpy(),
               front_s=g["front_s"][:n].cpu().numpy(), ap=int(g["pick"][0]), eo=int(g["pick"][1]),
               status=int(status.item()))
    return out


def check(g, ora_c, ora_e, ora_reach, tau, floor, idx=None):
    sel = slice(None) if idx is None else idx
    assert np.array_equal(g["correct"][sel], ora_c)
    assert np.array_equal(g["energy"][sel], ora_e)
    if ora_reach is not None and "reach" in g:
        assert np.array_equal(g["reach"][sel], ora_reach)
    ref = oracle.perf_graph(g["correct"], g["energy"], tau, floor)
    for k in ("front_c", "front_e", "front_s"):
        assert np.array_equal(g[k], ref[k]), k
    assert g["ap"] == ref["ap"] and g["eo"] == ref["eo"], (g["ap"], ref["ap"], g["eo"], ref["eo"])
    assert g["status"] == 0


def test_hand_graph(hs):
    d = json.load(open(os.path.join(GOLD, "hand_perf_graph.json")))
    conf = np.array(d["conf"], np.float32)
    ok = np.array(d["correct"], np.uint8)
    g = gpu_graph(hs, conf, ok, d["log2_bins"], d["weights"])
    assert g["correct"].tolist() == d["correct_by_b"] and g["energy"].tolist() == d["energy_by_b"]
    assert g["reach"].tolist() == d["reach_by_b"]
    assert g["front_c"].tolist() == d["front_c"] and g["front_s"].tolist() == d["front_s"]
    assert g["ap"] == d["ap"] and g["eo"] == d["eo"]
    assert g["model_correct"].tolist() == ok.sum(1).tolist()


def _case(rng, K, N, nan=True):
    conf = rng.random((K - 1, N)).astype(np.float32)
    conf[rng.random((K - 1, N)) < 0.1] = np.float32(1.0)
    conf[rng.random((K - 1, N)) < 0.05] = np.float32(0.0)
    if nan and N > 3:
        conf[0, 3] = np.nan
    ok = (rng.random((K, N)) < np.linspace(0.5, 0.9, K)[:, None]).astype(np.uint8)
    w = np.sort(rng.integers(1, 1000, size=K)).astype(np.int64)
    return conf, ok, w


@pytest.mark.parametrize("K,q,N", [(2, 4, 1), (2, 6, 2049), (3, 3, 4097), (4, 2, 1000), (5, 2, 3001),
                                   (6, 1, 777), (8, 1, 300), (3, 5, 9001), (4, 4, 2500)])
def test_whole_grid_vs_oracle(hs, K, q, N):
    rng = np.random.default_rng(100 + K * 10 + q)
    conf, ok, w = _case(rng, K, N)
    g = gpu_graph(hs, conf, ok, q, w)
    c, e, reach = oracle.replay(conf, ok, q, w)
    check(g, c, e, reach, int(ok[K - 1].sum()), int(ok[K - 2].sum()))


def test_explicit_vectors_and_host_tau(hs):
    rng = np.random.default_rng(7)
    conf, ok, w = _case(rng, 4, 5000)
    q = 6
    bv = rng.integers(0, (1 << q) + 2, size=(3000, 3)).astype(np.int32)
    g = gpu_graph(hs, conf, ok, q, w, bvecs=bv, tau=3000, floor=2500)
    c, e, reach = oracle.replay(conf, ok, q, w, bvecs=bv)
    check(g, c, e, reach, 3000, 2500)


def test_c2_validation_exhaustive_grid_sampled(hs):
    """The C2 validation workload at full size: 5 ViT stage models, 50,000
    samples, the GPU's confidences; the whole q = 4 grid (18^4 = 104,976
    vectors) on the GPU; 1,500 sampled vectors replayed by the oracle; the
    frontier / AP / EO recomputed by the oracle from the GPU's points."""
    fam = synth.FAMILIES["c2"]
    n = fam.n_val
    vids = np.arange(n, dtype=np.int64) + synth.VAL_ID_BASE
    lab = torch.from_numpy(synth.labels_np(fam.seed, vids, 1, fam.C).reshape(-1)).to(dev())
    xs = []
    for k in range(fam.K):
        bits = synth.fam_logits_np(fam, k, vids, "bf16", L=1, C=fam.C)
        xs.append(torch.from_numpy(bits.view(np.int16)).to(dev()).view(torch.bfloat16))
    r = hs.confidence_batched(xs, fam.temps, labels=lab)
    conf = r["conf"].view(fam.K, n)[: fam.K - 1].cpu().numpy()
    ok = r["correct"].view(fam.K, n).cpu().numpy()
    w = np.array([1, 2, 4, 8, 16], np.int64)        # ViT-XS .. ViT-L energy ratios (synthetic)
    q = 4
    g = gpu_graph(hs, conf, ok, q, w, reach=False)
    S = oracle.grid_size(fam.K, q)
    assert g["correct"].size == S
    idx = np.sort(np.random.default_rng(5).choice(S, 1500, replace=False))
    idx[0], idx[-1] = 0, S - 1
    bv = np.array([oracle.grid_vector(int(s), fam.K, q) for s in idx], np.int32)
    c, e, _ = oracle.replay(conf, ok, q, w, bvecs=bv)
    check(g, c, e, None, int(ok[-1].sum()), int(ok[-2].sum()), idx=idx)
    # the prefix-histogram path (whole grid) equals the direct replay of the same
    # vectors passed explicitly (two independent GPU paths)
    allv = np.array([oracle.grid_vector(int(s), fam.K, q) for s in range(S)], np.int32)
    gd = gpu_graph(hs, conf, ok, q, w, bvecs=allv, reach=False)
    assert np.array_equal(gd["correct"], g["correct"]) and np.array_equal(gd["energy"], g["energy"])
    # the exhaustive AP optimum never costs more than the greedy calibration (D5)
    cal = oracle.calibrate(conf, ok, q)
    cg, eg, _ = oracle.replay(conf, ok, q, w, bvecs=cal["b"][None, :])
    assert g["energy"][g["ap"]] <= eg[0] and g["correct"][g["ap"]] >= int(ok[-1].sum())
    # EO sits on the frontier with at least the second-largest model's accuracy
    assert g["correct"][g["eo"]] >= int(ok[-2].sum()) and g["eo"] in set(g["front_s"].tolist())


def test_graph_closed_forms_and_edges(hs):
    cs = np.arange(21, dtype=np.int64)
    kink = np.where(cs <= 10, cs, 10 + 5 * (cs - 10)).astype(np.int64)
    for C, E, tau, floor, ap, eo in ((cs, kink, 20, 0, 20, 10), (cs, kink, 20, 11, 20, 11),
                                     (cs, cs * cs, 20, 7, 20, 7),
                                     (np.array([2, 3]), np.array([4, 14]), 3, 0, 1, 1)):
        st = torch.zeros(1, dtype=torch.int32, device=dev())
        g = hs.perf_graph(torch.from_numpy(C).to(dev()), torch.from_numpy(E).to(dev()), 20,
                          tau=tau, floor=floor, status=st)
        torch.cuda.synchronize()
        assert g["pick"].tolist() == [ap, eo]
    # no points; one point; unreachable tau
    z = torch.zeros(0, dtype=torch.int64, device=dev())
    g = hs.perf_graph(z, z, 10, tau=3, floor=0)
    assert int(g["front_n"].item()) == 0 and g["pick"].tolist() == [-1, -1]
    one = torch.tensor([4], dtype=torch.int64, device=dev())
    g = hs.perf_graph(one, one * 3, 10, tau=5, floor=0)
    assert int(g["front_n"].item()) == 1 and g["pick"].tolist() == [-1, -1]
    # out-of-range points are ignored and flagged
    st = torch.zeros(1, dtype=torch.int32, device=dev())
    g = hs.perf_graph(torch.tensor([3, 11, 2], dtype=torch.int64, device=dev()),
                      torch.tensor([5, 1, -1], dtype=torch.int64, device=dev()), 10, tau=0, floor=0,
                      status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & 1 and int(g["front_n"].item()) == 1 and g["pick"].tolist() == [0, 0]


def test_router_offline_flow(hs):
    """The offline 'dataflow construction' through the Router: fit temperatures
    (Eq. 1), calibrate AP thresholds with them (Alg. 1 AP), build the threshold
    performance graph (AP / EO), then route -- each step checked against the oracle."""
    from paper_2505_12566_b200.router import Router
    fam = synth.scaled(synth.FAMILIES["c2"], n=4000, n_val=3000)
    dev_ = dev()
    vids = np.arange(fam.n_val, dtype=np.int64) + synth.VAL_ID_BASE
    lab = synth.labels_np(fam.seed, vids, 1, fam.C).reshape(-1)
    vbits = [synth.fam_logits_np(fam, k, vids, "bf16", L=1, C=fam.C) for k in range(fam.K)]
    val = [torch.from_numpy(b.view(np.int16)).to(dev_).view(torch.bfloat16) for b in vbits]
    labels = torch.from_numpy(lab).to(dev_)
    router = Router([hs.StageSpec(fam.C, 1.0) for _ in range(fam.K)], fam.n, fam.n_val, dev_,
                    log2_bins=fam.log2_bins)
    temps = router.fit_temperatures(val, labels)
    for k in range(fam.K):
        t_o = oracle.fit_temperature(vbits[k], lab, n_classes=fam.C)
        assert abs(temps[k] - t_o) <= 1e-5 * t_o
    cal = router.calibrate(val, labels)
    torch.cuda.synchronize()
    vconf = router.vconf.cpu().numpy()
    vok = router.vok.cpu().numpy()
    for k in range(fam.K - 1):                   # the fitted T are the ones used
        ref = oracle.confidence(vbits[k], fam.n_val, 1, fam.C, fam.C, temps[k], labels=lab)
        assert np.max(np.abs(vconf[k] - ref["conf"]) / ref["conf"]) <= 1e-5
    assert cal["b"].cpu().numpy().tolist() == oracle.calibrate(vconf, vok, fam.log2_bins)["b"].tolist()
    w = [1, 2, 4, 8, 16]
    g = router.performance_graph(w, log2_bins=3)
    c, e, _ = oracle.replay(vconf, vok, 3, w)
    ref = oracle.perf_graph(c, e, int(vok[-1].sum()), int(vok[-2].sum()))
    assert g["front_s"].numpy().tolist() == ref["front_s"].tolist()
    assert g["ap"]["b"] == oracle.grid_vector(ref["ap"], fam.K, 3)
    assert g["eo"]["b"] == oracle.grid_vector(ref["eo"], fam.K, 3)
    assert g["ap"]["correct"] >= int(vok[-1].sum())
    # route with the AP thresholds of the graph (host list) and with the calibrated ones
    ids = np.arange(fam.n, dtype=np.int64)
    logits = [torch.from_numpy(synth.fam_logits_np(fam, k, ids, "bf16", L=1, C=fam.C)
                               .view(np.int16)).to(dev_).view(torch.bfloat16) for k in range(fam.K)]
    router.route(logits, thresholds=g["ap"]["t"])
    res = router.cascade.results()
    assert sum(r["n_acc"] for r in res) == fam.n
