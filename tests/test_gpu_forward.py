"""GPU checks of the multi-GPU exchange over peer memory (hs_peer_*, SURVEY
8(e)): W virtual ranks on ONE GPU, each with its own peer region,
addressed through the same hs_peer_t pointer tables a real multi-GPU group
builds from CUDA IPC mappings (dist.PeerGroup.local_group).

* forwarding: after publish -> scatter -> wait, every destination rank holds
  exactly its contiguous block of the GLOBAL stable deferred list (rank-major
  concatenation of the per-rank lists given by the oracle's stable split,
  P:443-444), with its payload rows; the regions are reused over several
  forwards (device epochs, re-armed completion counter, alternating sets).
* calibration: every virtual rank runs hs_calibrate_thresholds_peer on its
  shard of a validation set (one stream per rank, so the W cooperative kernels
  run side by side) and must select exactly the thresholds the oracle selects
  on the WHOLE set (the pushed histograms are summed inside the kernel).
* the comm-aware cascade step (hs_cascade_step_peer) over W virtual ranks
  equals the oracle's cascade of the whole batch."""
import numpy as np
import pytest
import torch

import oracle
from paper_2505_12566_b200 import dist as hsd

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hs(libhs):
    return libhs


def _payload_of(ids: np.ndarray, P: int) -> np.ndarray:
    return ((ids[:, None] * 7 + np.arange(P)[None, :]) % 251).astype(np.uint8)


def _expected_blocks(conf_all, bounds, t, dest, world):
    glob = np.concatenate([bounds[g] + oracle.route(conf_all[bounds[g]:bounds[g + 1]], t, False)[1]
                           for g in range(world)]).astype(np.int64)
    lo_b = hsd.block_bounds(len(glob), len(dest))
    return [np.concatenate([glob[lo_b[i]:lo_b[i + 1]] for i, h in enumerate(dest) if h == g] or
                           [np.zeros(0, np.int64)]) for g in range(world)]


@pytest.mark.parametrize("world,dest,P,fused", [
    (1, None, 16, False), (2, None, 0, False), (3, None, 32, False), (3, [2], 16, False),
    (4, [0, 2], 0, False), (8, [7, 1, 4], 48, False), (8, None, 0, False),
    (1, None, 16, True), (2, None, 0, True), (3, None, 32, True), (4, None, 16, True), (8, None, 0, True)])
def test_peer_forward_virtual_ranks(hs, world, dest, P, fused):
    """fused=False: the three phases for all ranks in turn on one stream;
    fused=True: hs_peer_forward per rank on its own stream (the kernels of the
    ranks run side by side and synchronise through the flags).  The fused
    variant needs every virtual rank's spinning scatter grid resident at once on
    the one GPU, so it runs the balanced cases with small grids (on a real
    group each GPU runs only its own rank's kernels)."""
    dev = torch.device("cuda:0")
    n = 6001
    rng = np.random.default_rng(world * 10 + P)
    conf_all = rng.random(n).astype(np.float32)
    destl = list(range(world)) if dest is None else dest
    bounds = [g * n // world for g in range(world + 1)]
    cap = max(bounds[g + 1] - bounds[g] for g in range(world))
    if dest is not None:
        cap = n      # placed blocks can exceed a rank's shard
    grp = hsd.PeerGroup.local_group(world, cap, P, 12, K=8, device=dev)
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    for st_ in streams:
        st_.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    for it, t in enumerate((0.6, 0.25, 0.97, 0.0, 0.5, 1.0)):
        outs = []
        for g in range(world):
            lo, hi = bounds[g], bounds[g + 1]
            ids = torch.arange(lo, hi, dtype=torch.int64, device=dev)
            pay = torch.from_numpy(_payload_of(np.arange(lo, hi), P)).to(dev) if P else None
            outs.append(hs.route_compact(torch.from_numpy(conf_all[lo:hi]).to(dev), t, ids=ids, payload=pay))
        torch.cuda.synchronize()
        st = it % 2
        rc = [grp[g].recv_count[it:it + 1] for g in range(world)]
        if fused:
            for g in range(world):
                hs.peer_forward(grp[g].g, st, outs[g]["def_ids"], outs[g]["counts"][1:2], rc[g],
                                payload=outs[g].get("def_payload"), dest_ranks=dest,
                                status=grp[g].status, stream=streams[g])
        else:
            for g in range(world):
                hs.peer_forward_publish(grp[g].g, outs[g]["counts"][1:2], status=grp[g].status)
            for g in range(world):
                hs.peer_forward_scatter(grp[g].g, st, outs[g]["def_ids"], rc[g],
                                        payload=outs[g].get("def_payload"), dest_ranks=dest,
                                        status=grp[g].status)
            for g in range(world):
                hs.peer_forward_wait(grp[g].g, status=grp[g].status)
        torch.cuda.synchronize()
        want = _expected_blocks(conf_all, bounds, t, destl, world)
        for g in range(world):
            assert int(grp[g].status.item()) == 0
            got_n = int(rc[g].item())
            assert got_n == len(want[g]), (it, g)
            assert np.array_equal(grp[g].recv_ids(st)[:got_n].cpu().numpy(), want[g]), (it, g)
            if P:
                got_p = grp[g].recv_payload(st)[:got_n].cpu().numpy()
                assert np.array_equal(got_p, _payload_of(want[g], P)), (it, g)
    grp[0].close()


def test_peer_forward_argument_errors(hs):
    dev = torch.device("cuda:0")
    grp = hsd.PeerGroup.local_group(2, 16, 0, 12, device=dev)
    c = torch.zeros(2, dtype=torch.int64, device=dev)
    with pytest.raises(hs.HsError):
        hs.peer_forward(grp[0].g, 2, c, c[:1], c[1:])                     # set outside {0, 1}
    with pytest.raises(hs.HsError):
        hs.peer_forward(grp[0].g, 0, c, c[:1], c[1:], dest_ranks=[1, 1])  # repeated destination
    with pytest.raises(hs.HsError):
        hs.peer_forward(grp[0].g, 0, c, c[:1], c[1:], payload=c)          # regions sized without payload
    bad = hsd.PeerGroup.local_group(2, 16, 0, 12, device=dev)[0].g
    bad.world = 9
    with pytest.raises(hs.HsError):
        hs.peer_forward(bad, 0, c, c[:1], c[1:])
    grp[0].close()


def test_peer_forward_times_out_instead_of_hanging(hs):
    """A peer that never publishes: the scatter and wait kernels give up after
    10 s, flag STATUS_TIMEOUT, receive nothing (the GPU is not hung); the
    completion counter is re-armed, so a later forward works."""
    dev = torch.device("cuda:0")
    grp = hsd.PeerGroup.local_group(2, 8, 0, 12, device=dev)
    ids = torch.arange(4, dtype=torch.int64, device=dev)
    cnt = torch.tensor([4], dtype=torch.int64, device=dev)
    rc = grp[0].recv_count[:1]
    hs.peer_forward(grp[0].g, 0, ids, cnt, rc, status=grp[0].status)      # rank 1 never publishes
    torch.cuda.synchronize()
    assert int(grp[0].status.item()) & hs.STATUS_TIMEOUT
    assert int(rc.item()) == 0


def _calib_case(seed, n, K):
    rng = np.random.default_rng(seed)
    d = rng.uniform(size=n)
    ok = np.stack([(d + 0.3 * rng.normal(size=n) < 0.5 + 0.08 * k) for k in range(K)]).astype(np.uint8)
    conf = np.clip(np.where(ok[:K - 1] == 1, rng.beta(5, 2, (K - 1, n)), rng.beta(2, 3, (K - 1, n))),
                   0, 1).astype(np.float32)
    conf[0, :: 97] = 1.0
    return conf, ok


@pytest.mark.parametrize("world,n,q,K", [(1, 3000, 12, 5), (2, 7000, 12, 5), (3, 9001, 10, 4),
                                         (4, 20000, 12, 5), (8, 16000, 8, 3), (2, 1, 4, 2)])
def test_peer_calibration_equals_oracle_on_the_whole_set(hs, world, n, q, K):
    dev = torch.device("cuda:0")
    conf, ok = _calib_case(world * 100 + n, n, K)
    ref = oracle.calibrate(conf.astype(np.float64), ok, q)
    grp = hsd.PeerGroup.local_group(world, 16, 0, q, device=dev)
    bounds = [g * n // world for g in range(world + 1)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    for st_ in streams:
        st_.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    outs = []
    for rep in range(3):                 # regions reused: round counters advance
        outs = []
        for g in range(world):
            lo, hi = bounds[g], bounds[g + 1]
            c = torch.from_numpy(np.ascontiguousarray(conf[:, lo:hi])).to(dev)
            o = torch.from_numpy(np.ascontiguousarray(ok[:, lo:hi])).to(dev)
            outs.append((c, o))
        torch.cuda.synchronize()
        res = [hs.calibrate_thresholds_peer(outs[g][0], outs[g][1], grp[g].g, log2_bins=q,
                                            status=grp[g].status, stream=streams[g])
               for g in range(world)]
        torch.cuda.synchronize()
        for g in range(world):
            assert int(grp[g].status.item()) == 0
            assert np.array_equal(res[g]["b"].cpu().numpy(), ref["b"]), (rep, g)
            assert int(res[g]["correct_total"].item()) == ref["correct_total"]
            assert np.array_equal(res[g]["reach"].cpu().numpy(), ref["reach"])
            assert np.array_equal(res[g]["handled"].cpu().numpy(), ref["handled"])
    grp[0].close()


@pytest.mark.parametrize("world,placed", [(1, False), (2, False), (4, False), (2, True)])
def test_peer_cascade_step_equals_oracle_cascade(hs, world, placed):
    """The comm-aware cascade step over W virtual ranks (balanced placement):
    the union of the accepted lists of stage k over all ranks equals the
    oracle's stage-k list of the whole batch (a request's stage does not
    depend on where it was routed)."""
    from workload import synth
    dev = torch.device("cuda:0")
    fam = synth.scaled(synth.FAMILIES["c2"], n=3000)
    K, n, C = fam.K, fam.n, fam.C
    ids_all = np.arange(n, dtype=np.int64)
    logits = [torch.from_numpy(synth.fam_logits_np(fam, k, ids_all).view(np.int16)).to(dev).view(torch.bfloat16)
              for k in range(K)]
    t = [float(np.float32(x)) for x in (0.55, 0.3, 0.6, 0.45, 0.0)]
    conf = np.stack([oracle.confidence(logits[k].view(torch.int16).cpu().numpy().view(np.uint16), n, 1, C, C,
                                       fam.temps[k])["conf"] for k in range(K)])
    stage_of = oracle.cascade(conf, np.array(t, np.float64))
    near = np.zeros(n, bool)
    for k in range(K - 1):
        near |= np.abs(conf[k] - t[k]) <= 1e-5 * t[k]
    bounds = [g * n // world for g in range(world + 1)]
    cap = max(bounds[g + 1] - bounds[g] for g in range(world))
    next_ranks = None
    if placed:       # replicas by the zero-queuing rule: a rank may receive every deferral
        ranks = hsd.placed_ranks(world, hsd.replica_counts(world, [1, .5, .3, .2, .2], [1, 2, 4, 8, 16]))
        next_ranks = ranks[1:]
        cap = world * cap
    grp = hsd.PeerGroup.local_group(world, cap, 0, 12, K=K, device=dev)
    casc = [__import__("paper_2505_12566_b200").Cascade(cap, [
        __import__("paper_2505_12566_b200").StageSpec(C, fam.temps[k]) for k in range(K)], dev)
        for _ in range(world)]
    thr = torch.tensor(t, dtype=torch.float32, device=dev)
    ids = [torch.arange(bounds[g], bounds[g + 1], dtype=torch.int64, device=dev) for g in range(world)]
    streams = [torch.cuda.Stream(device=dev) for _ in range(world)]
    for st_ in streams:
        st_.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    for g in range(world):
        casc[g].route(logits, thr, n=bounds[g + 1] - bounds[g], ids=ids[g], by_id=True, peer=grp[g],
                      next_ranks=next_ranks, stream=streams[g])
    torch.cuda.synchronize()
    for k in range(K):
        got = np.sort(np.concatenate([casc[g].results()[k]["ids"].numpy() for g in range(world)]))
        want = np.flatnonzero(stage_of == k)
        assert np.array_equal(got[~near[got]], want[~near[want]]), k
    assert all(int(grp[g].status.item()) == 0 for g in range(world))
    grp[0].close()
