"""GPU check of the peer-memory forwarding of deferred requests (hs_forward_*,
SURVEY 8(e) v2): W virtual ranks on ONE GPU, each with its own count / done
arrays and receive buffers, addressed through the same pointer tables a real
multi-GPU group builds from CUDA IPC mappings.  After publish -> scatter ->
wait, every destination rank must hold exactly its contiguous block of the
GLOBAL stable deferred list (rank-major concatenation of the per-rank lists
given by the oracle's stable split), with its payload rows; the same
buffers are reused for a second forward (epochs, re-armed counter)."""
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


@pytest.mark.parametrize("world,dest,P", [(1, None, 16), (2, None, 0), (3, None, 32), (3, [2], 16),
                                          (4, [0, 2], 0), (8, [7, 1, 4], 48)])
def test_peer_forward_virtual_ranks(hs, world, dest, P):
    dev = torch.device("cuda:0")
    n = 6001
    rng = np.random.default_rng(world * 10 + P)
    conf_all = rng.random(n).astype(np.float32)
    dest = list(range(world)) if dest is None else dest
    bounds = [g * n // world for g in range(world + 1)]
    cap = max(bounds[g + 1] - bounds[g] for g in range(world))
    counts = [torch.zeros(world, dtype=torch.int64, device=dev) for _ in range(world)]
    done = [torch.zeros(world, dtype=torch.int64, device=dev) for _ in range(world)]
    recv_ids = [torch.full((world * cap,), -1, dtype=torch.int64, device=dev) for _ in range(world)]
    recv_pay = [torch.zeros(world * cap * max(P, 16), dtype=torch.uint8, device=dev) for _ in range(world)]
    wss = [torch.zeros(256, dtype=torch.uint8, device=dev) for _ in range(world)]
    rcnt = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    for epoch, t in ((1, 0.6), (2, 0.25), (3, 0.97), (4, 0.0), (5, 0.5)):
        outs = []
        for g in range(world):
            lo, hi = bounds[g], bounds[g + 1]
            ids = torch.arange(lo, hi, dtype=torch.int64, device=dev)
            pay = torch.from_numpy(_payload_of(np.arange(lo, hi), P)).to(dev) if P else None
            o = hs.route_compact(torch.from_numpy(conf_all[lo:hi]).to(dev), t, ids=ids, payload=pay)
            outs.append(o)
        for g in range(world):
            hs.forward_publish(outs[g]["counts"][1:2], cap, g, [c.data_ptr() for c in counts], epoch)
        for g in range(world):
            hs.forward_scatter(outs[g]["def_ids"], cap, g, counts[g], [d.data_ptr() for d in done],
                               [r.data_ptr() for r in recv_ids], dest, epoch, rcnt[g], wss[g],
                               payload=outs[g].get("def_payload"), payload_row_bytes=P,
                               peer_recv_payload=[r.data_ptr() for r in recv_pay] if P else None)
        for g in range(world):
            hs.forward_wait(done[g], world, epoch)
        torch.cuda.synchronize()
        # expected: the oracle's per-rank stable deferred lists, concatenated, split into blocks
        glob = np.concatenate([bounds[g] + oracle.route(conf_all[bounds[g]:bounds[g + 1]], t, False)[1]
                               for g in range(world)]).astype(np.int64)
        lo_b = hsd.block_bounds(len(glob), len(dest))
        for g in range(world):
            want = np.concatenate([glob[lo_b[i]:lo_b[i + 1]] for i, h in enumerate(dest) if h == g] or
                                  [np.zeros(0, np.int64)])
            got_n = int(rcnt[g].item())
            assert got_n == len(want), (epoch, g)
            assert np.array_equal(recv_ids[g][:got_n].cpu().numpy(), want), (epoch, g)
            if P:
                got_p = recv_pay[g][: got_n * P].cpu().numpy().reshape(got_n, P)
                assert np.array_equal(got_p, _payload_of(want, P)), (epoch, g)
        assert all(int(w.sum()) == 0 for w in wss)              # completion counters re-armed
        assert all((c.cpu().numpy() >> 32 == epoch).all() for c in counts)


def test_forward_argument_errors(hs):
    dev = torch.device("cuda:0")
    c = torch.zeros(2, dtype=torch.int64, device=dev)
    ws = torch.zeros(256, dtype=torch.uint8, device=dev)
    with pytest.raises(hs.HsError):
        hs.forward_publish(c[:1], 10, 0, [c.data_ptr()] * 2, 0)          # epoch 0
    with pytest.raises(hs.HsError):
        hs.forward_scatter(c, 10, 0, c, [c.data_ptr()] * 2, [c.data_ptr()] * 2, [1, 1], 1, c[:1], ws)
    with pytest.raises(hs.HsError):
        hs.forward_wait(c, 9, 1)


def test_forward_times_out_instead_of_hanging(hs):
    """A peer that never publishes: the scatter and wait kernels give up after
    10 s, flag STATUS_TIMEOUT and write nothing (the GPU is not hung)."""
    dev = torch.device("cuda:0")
    W = 2
    counts = [torch.zeros(W, dtype=torch.int64, device=dev) for _ in range(W)]
    done = [torch.zeros(W, dtype=torch.int64, device=dev) for _ in range(W)]
    recv = [torch.full((8,), -7, dtype=torch.int64, device=dev) for _ in range(W)]
    ws = torch.zeros(256, dtype=torch.uint8, device=dev)
    st = torch.zeros(1, dtype=torch.int32, device=dev)
    rc = torch.zeros(1, dtype=torch.int64, device=dev)
    ids = torch.arange(4, dtype=torch.int64, device=dev)
    cnt = torch.tensor([4], dtype=torch.int64, device=dev)
    hs.forward_publish(cnt, 4, 0, [c.data_ptr() for c in counts], 1)      # rank 1 never publishes
    hs.forward_scatter(ids, 4, 0, counts[0], [d.data_ptr() for d in done], [r.data_ptr() for r in recv],
                       [0, 1], 1, rc, ws, status=st)
    hs.forward_wait(done[0], W, 1, status=st)
    torch.cuda.synchronize()
    assert int(st.item()) & hs.STATUS_TIMEOUT
    assert (recv[0] == -7).all() and (recv[1] == -7).all()
