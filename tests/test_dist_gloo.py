"""Multi-rank host logic on CPU (gloo, world size 2 and 3): the exchange plan and
the forwarding of deferred requests reproduce the oracle's GLOBAL stable
deferred list, split into contiguous blocks over the next stage's ranks."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
from paper_2505_12566_b200 import dist as hsd


def test_exchange_plan_blocks():
    counts = [5, 0, 7, 3]
    plan = hsd.exchange_plan(counts, [0, 1, 2, 3], 4)
    assert [sum(r) for r in plan] == counts                         # everything is sent
    recv = [sum(plan[g][h] for g in range(4)) for h in range(4)]
    lo = hsd.block_bounds(15, 4)
    assert recv == [lo[i + 1] - lo[i] for i in range(4)]            # contiguous blocks
    plan = hsd.exchange_plan(counts, [2], 4)                         # one replica of m_{k+1}
    assert all(plan[g][2] == counts[g] for g in range(4))
    assert hsd.exchange_plan([0, 0], [0, 1], 2) == [[0, 0], [0, 0]]
    assert hsd.global_order_offsets(counts) == [0, 5, 5, 12]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, conf_all, t, dest, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n = conf_all.shape[0]
    lo, hi = rank * n // world, (rank + 1) * n // world
    # this rank's stage decision (the oracle stands in for the GPU kernels here)
    acc, dfr = oracle.route(conf_all[lo:hi], t, False)
    ids = torch.arange(lo, hi, dtype=torch.int64)[torch.from_numpy(dfr)]
    payload = (ids.view(-1, 1) * 3 + torch.arange(4).view(1, 4)).to(torch.int32)
    buf = torch.full((hi - lo,), -1, dtype=torch.int64)
    buf[: len(ids)] = ids
    pbuf = torch.zeros(hi - lo, 4, dtype=torch.int32)
    pbuf[: len(ids)] = payload
    cnt = torch.tensor([len(ids)], dtype=torch.int64)
    out_ids, out_pay, n_recv = hsd.forward_deferred(buf, cnt, dest_ranks=dest, payload=pbuf)
    q.put((rank, out_ids.tolist(), out_pay.tolist(), n_recv))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,dest", [(2, None), (3, None), (3, [2]), (3, [0, 2])])
def test_forward_deferred_matches_global_order(world, dest):
    rng = np.random.default_rng(world)
    n = 1000
    conf = rng.uniform(size=n)
    t = 0.6
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, conf, t, dest, q)) for r in range(world)]
    for p in procs:
        p.start()
    got = dict()
    for _ in range(world):
        r, ids, pay, nr = q.get(timeout=120)
        got[r] = (ids, pay, nr)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    _, dfr_global = oracle.route(conf, t, False)      # global stable deferred list
    dest_ranks = list(range(world)) if dest is None else dest
    lo = hsd.block_bounds(len(dfr_global), len(dest_ranks))
    cat = []
    for i, h in enumerate(dest_ranks):
        ids, pay, nr = got[h]
        assert ids == list(dfr_global[lo[i]:lo[i + 1]])
        assert pay == [[3 * x + j for j in range(4)] for x in ids]
        cat += ids
    assert cat == list(dfr_global)
    for h in range(world):
        if h not in dest_ranks:
            assert got[h][2] == 0


def test_bench_spawns_ranks_and_reduces():
    """bench.py --gpus 2 without a torchrun environment re-launches itself as
    two ranks (torch.distributed.run, 127.0.0.1 rendezvous); the ranks join a
    gloo group, exchange handles once and reduce with max / sum over ranks --
    the host side of the multi-GPU bench, on CPU."""
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK", "LOCAL_RANK")}
    r = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--gpus", "2", "--plumbing-check"],
                       capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads(r.stdout.strip().splitlines()[-1])
    assert line == {"plumbing_check": True, "world": 2, "handles_ok": True, "max": [1.0, 10.0],
                    "sum": [3.0]}


def test_replica_counts_follow_the_zero_queuing_rule():
    """R_m proportional to rho_m l_m, rounded to positive integers,
    and the world's GPUs shared out exactly."""
    R = hsd.replica_counts(8, [1.0, 0.5, 0.3, 0.2, 0.18], [1, 2, 4, 8, 16])
    assert sum(R) == 8 and min(R) >= 1
    w = [1.0 * 1, 0.5 * 2, 0.3 * 4, 0.2 * 8, 0.18 * 16]
    assert R[4] == max(R) and R[4] >= R[0]          # the giant model carries the most load
    # exact proportions are reproduced when they are integers
    assert hsd.replica_counts(6, [1, 1, 1], [1, 2, 3]) == [1, 2, 3]
    assert hsd.replica_counts(4, [1, 0, 0], [1, 1, 1]) == [2, 1, 1]     # every model keeps a replica
    assert hsd.replica_counts(2, [1, 1, 1], [1, 1, 1]) == [1, 1, 1]     # more models than GPUs
    assert hsd.replica_counts(8, [0, 0], [1, 1]) == [1, 1]
    ranks = hsd.placed_ranks(8, R)
    assert [len(r) for r in ranks] == R
    assert sorted(x for r in ranks for x in r) == list(range(8))       # every GPU used once
    assert hsd.placed_ranks(3, [2, 2]) == [[0, 1], [2, 0]]
