"""The library's NCCL communicator (hs_comm_*) and the request-sharded
calibration built on it (hs_calibrate_thresholds_comm), at world size 1 on one
B200 (the all-reduce runs; with one rank it is the identity): bit-exact with
the single-GPU calibration and the oracle (integer algorithm, D5)."""
import numpy as np
import pytest
import torch

import oracle
from workload import synth

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


@pytest.mark.parametrize("K,N,q", [(2, 4096, 12), (5, 50000, 12), (3, 777, 4)])
def test_calibrate_comm_world1_bit_exact(hs, K, N, q):
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(K * 1000 + N)
    conf = rng.random((K - 1, N)).astype(np.float32)
    conf[0, :5] = np.nan
    ok = (rng.random((K, N)) < np.linspace(0.6, 0.9, K)[:, None]).astype(np.uint8)
    c = torch.from_numpy(conf).to(dev)
    o = torch.from_numpy(ok).to(dev)
    comm = hs.comm_create(hs.comm_unique_id(), 0, 1, 0)
    try:
        a = hs.calibrate_thresholds_comm(c, o, comm, log2_bins=q)
        b = hs.calibrate_thresholds_comm(c, o, None, log2_bins=q)
        r = hs.calibrate_thresholds(c, o, log2_bins=q)
        torch.cuda.synchronize()
    finally:
        hs.comm_destroy(comm)
    ref = oracle.calibrate(conf, ok, q)
    for out in (a, b, r):
        assert out["b"].cpu().numpy().tolist() == ref["b"].tolist()
        assert out["reach"].cpu().numpy().tolist() == ref["reach"].tolist()
        assert out["handled"].cpu().numpy().tolist() == ref["handled"].tolist()
        assert int(out["correct_total"].item()) == ref["correct_total"]
        assert np.array_equal(out["t"].cpu().numpy(), r["t"].cpu().numpy())


def test_router_native_comm(hs):
    from paper_2505_12566_b200.router import Router
    dev = torch.device("cuda:0")
    fam = synth.scaled(synth.FAMILIES["c2"], n=2000, n_val=5000)
    vids = np.arange(fam.n_val, dtype=np.int64) + synth.VAL_ID_BASE
    labels = torch.from_numpy(synth.labels_np(fam.seed, vids, 1, fam.C).reshape(-1)).to(dev)
    val = [torch.from_numpy(synth.fam_logits_np(fam, k, vids, "bf16", L=1, C=fam.C).view(np.int16))
           .to(dev).view(torch.bfloat16) for k in range(fam.K)]
    stages = [hs.StageSpec(fam.C, fam.temps[k]) for k in range(fam.K)]
    r1 = Router(stages, fam.n, fam.n_val, dev, log2_bins=fam.log2_bins)
    r2 = Router(stages, fam.n, fam.n_val, dev, log2_bins=fam.log2_bins, native_comm=True)
    a = r1.calibrate(val, labels)
    b = r2.calibrate(val, labels)
    torch.cuda.synchronize()
    assert a["b"].cpu().tolist() == b["b"].cpu().tolist()
    assert a["t"].cpu().tolist() == b["t"].cpu().tolist()
    hs.comm_destroy(r2.hs_comm)


def test_forward_nccl_world1(hs):
    """hs_forward_nccl at world size 1 (self send / receive through NCCL): the
    receiver gets the whole deferred list, with payload, in order."""
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(3)
    conf = torch.from_numpy(rng.random(5000).astype(np.float32)).to(dev)
    ids = torch.arange(100, 5100, dtype=torch.int64, device=dev)
    pay = torch.from_numpy(rng.integers(0, 255, (5000, 32)).astype(np.uint8)).to(dev)
    o = hs.route_compact(conf, 0.6, ids=ids, payload=pay)
    comm = hs.comm_create(hs.comm_unique_id(), 0, 1, 0)
    try:
        rid, rpay, n = hs.forward_nccl(o["def_ids"], o["counts"][1:2], comm, 1, payload=o["def_payload"],
                                       payload_row_bytes=32)
        torch.cuda.synchronize()
    finally:
        hs.comm_destroy(comm)
    c = conf.cpu().numpy()
    want = np.flatnonzero(~(c >= np.float32(0.6))) + 100
    assert n == len(want) and np.array_equal(rid.cpu().numpy(), want)
    assert np.array_equal(rpay.cpu().numpy().reshape(n, 32), pay.cpu().numpy()[want - 100])


@pytest.mark.parametrize("K,N,q,passes", [(3, 4000, 6, 2), (5, 20000, 12, 1), (4, 999, 3, 3)])
def test_calibrate_comm_refinement_world1(hs, K, N, q, passes):
    """hs_calibrate_thresholds_comm_ex with refinement passes (the histogram and
    A_k all-reduced per pass and stage, the replay counts all-reduced) equals
    the oracle's refinement at world size 1 -- with the communicator and
    without -- and the single-GPU call."""
    dev = torch.device("cuda:0")
    rng = np.random.default_rng(K * 77 + N)
    d = rng.random(N)
    ok = np.stack([(d + 0.3 * rng.normal(size=N) < 0.5 + 0.1 * k) for k in range(K)]).astype(np.uint8)
    conf = np.clip(np.where(ok[:K - 1] == 1, rng.beta(5, 2, (K - 1, N)), rng.beta(2, 3, (K - 1, N))),
                   0, 1).astype(np.float32)
    c = torch.from_numpy(conf).to(dev)
    o = torch.from_numpy(ok).to(dev)
    comm = hs.comm_create(hs.comm_unique_id(), 0, 1, 0)
    try:
        a = hs.calibrate_thresholds_comm(c, o, comm, log2_bins=q, refine_passes=passes)
        b = hs.calibrate_thresholds_comm(c, o, None, log2_bins=q, refine_passes=passes)
        r = hs.calibrate_thresholds(c, o, log2_bins=q, refine_passes=passes)
        torch.cuda.synchronize()
    finally:
        hs.comm_destroy(comm)
    ref = oracle.calibrate(conf.astype(np.float64), ok, q, refine_passes=passes)
    for out in (a, b, r):
        assert out["b"].cpu().numpy().tolist() == ref["b"].tolist()
        assert out["reach"].cpu().numpy().tolist() == ref["reach"].tolist()
        assert out["handled"].cpu().numpy().tolist() == ref["handled"].tolist()
        assert int(out["correct_total"].item()) == ref["correct_total"]
