"""The multi-GPU cascade with REAL processes: W ranks, one process each, joined
by CUDA IPC mappings of their peer regions (dist.PeerGroup) -- the path the
8-GPU bench runs -- here all on cuda:0 (the processes time-slice the one GPU
of this pool; the exchange goes through the same IPC-mapped memory and
system-scope flags).  torch.distributed (gloo) is used only to exchange the
IPC handles once and to collect the results.

Checked against the oracle on the WHOLE job:
  * calibration: every rank selects the b_k the oracle's D5 sweep selects on
    the union of the ranks' validation shards (GPU confidences, check (i));
  * routing (balanced placement, dense stage batches): the union over ranks
    of each stage's accepted ids equals the oracle's stage list of the whole
    batch under those thresholds, near-threshold requests (G18) excluded and
    counted; a rank's stage-k batch is its contiguous block of the global
    stable deferred list."""
import os
import socket

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

REL = 1e-5


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, n, n_val, graph, q, placed=False):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2505_12566_b200 as hs
        import workload
        from paper_2505_12566_b200 import dist as hsd
        from paper_2505_12566_b200.router import Router
        from workload import synth
        dev = torch.device("cuda:0")
        torch.cuda.set_device(dev)
        fam = synth.scaled(synth.FAMILIES["c2"], n=n, n_val=n_val)
        K = fam.K
        val = []
        for k in range(K):
            v = torch.empty(n_val, fam.C, dtype=torch.bfloat16, device=dev)
            workload.gpu_logits(v, fam, k, n=n_val, id_base=synth.VAL_ID_BASE + rank * n_val)
            val.append(v)
        lab = torch.empty(n_val, dtype=torch.int32, device=dev)
        workload.gpu_labels(lab, fam, id_base=synth.VAL_ID_BASE + rank * n_val, n=n_val)
        cap = n * (world if placed else 1)
        peer = hsd.PeerGroup(cap, 0, fam.log2_bins, K=K, device=dev)
        stages = [hs.StageSpec(fam.C, fam.temps[k]) for k in range(K)]
        router = Router(stages, cap, n_val, dev, log2_bins=fam.log2_bins, peer=peer)
        if placed:      # model m's replicas on placed ranks: every deferral to one rank
            router.next_ranks = hsd.placed_ranks(world, hsd.replica_counts(
                world, [1, .5, .3, .2, .2], [1, 2, 4, 8, 16]))[1:]
        ids0 = torch.arange(rank * n, (rank + 1) * n, dtype=torch.int64, device=dev)
        x0 = torch.empty(n, fam.C, dtype=torch.bfloat16, device=dev)
        workload.gpu_logits(x0, fam, 0, id_base=rank * n, n=n)
        # dense stage batches, discovered stage by stage (as bench.py does)
        router.calibrate(val, lab)
        logits = [x0] + [None] * (K - 1)
        for k in range(1, K):
            router.route(logits, n=n, ids=ids0, by_id=False, upto=k - 1)
            torch.cuda.synchronize()
            nk = int(peer.recv_count[k - 1].item())
            x = torch.empty(max(nk, 1), fam.C, dtype=torch.bfloat16, device=dev)
            if nk:
                workload.gpu_logits(x, fam, k, ids=peer.recv_ids((k - 1) % 2)[:nk].clone(), n=nk)
            logits[k] = x
        s = torch.cuda.Stream(device=dev)
        s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far

        def step():
            router.calibrate(val, lab)
            router.route(logits, n=n, ids=ids0, by_id=False, overlap_first=True)

        with torch.cuda.stream(s):
            step()
            if graph:
                s.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    step()
                g.replay()
                g.replay()
        torch.cuda.synchronize()
        res = router.cascade.results()
        out = {"rank": rank, "status": int(router.status.item()) | int(peer.status.item()),
               "b": router.cal["b"].cpu().tolist(), "t": router.cal["t"].cpu().tolist(),
               "vconf": router.vconf.cpu().numpy(), "vok": router.vok.cpu().numpy(),
               "acc": [r["ids"].numpy() for r in res],
               "recv": [int(x) for x in peer.recv_count[: K - 1].cpu().tolist()]}
        q.put(out)
        dist.barrier()
        peer.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,graph,placed", [(2, False, False), (2, True, False), (3, True, False),
                                                (3, True, True)])
def test_peer_group_across_processes_equals_oracle(libhs, world, graph, placed):
    import torch.multiprocessing as mp
    import oracle
    from paper_2505_12566_b200 import dist as hsd
    from workload import synth
    n, n_val = 4000, 3000
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n, n_val, graph, q, placed))
             for r in range(world)]
    for p in procs:
        p.start()
    outs = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    outs.sort(key=lambda o: o["rank"])
    fam = synth.scaled(synth.FAMILIES["c2"], n=n, n_val=n_val)
    K = fam.K
    assert all(o["status"] == 0 for o in outs)
    # calibration: identical on every rank, equal to the oracle on the union (check (i))
    vconf = np.concatenate([o["vconf"] for o in outs], axis=1)
    vok = np.concatenate([o["vok"] for o in outs], axis=1)
    ref = oracle.calibrate(vconf, vok, fam.log2_bins)
    for o in outs:
        assert o["b"] == ref["b"].tolist()
    t = np.array(outs[0]["t"], np.float64)
    # routing of the whole job
    ids = np.arange(world * n, dtype=np.int64)
    conf = np.stack([oracle.confidence(synth.fam_logits_np(fam, k, ids), len(ids), 1, fam.C, fam.C,
                                       fam.temps[k])["conf"] for k in range(K)])
    stage_of = oracle.cascade(conf, t)
    near = np.zeros(len(ids), bool)
    per = []
    for k in range(K - 1):
        nk = (stage_of >= k) & (np.abs(conf[k] - t[k]) <= REL * t[k])
        per.append(int(nk.sum()))
        near |= nk
    print(f"world {world}: near-threshold requests per stage {per}")
    for k in range(K):
        got = np.sort(np.concatenate([o["acc"][k] for o in outs]))
        want = np.flatnonzero(stage_of == k)
        assert np.array_equal(got[~near[got]], want[~near[want]]), k
    # balanced placement: rank g received block g of the global deferred list
    for k in range(K - 1 if not placed else 0):
        D = int((stage_of > k).sum())
        lo = hsd.block_bounds(D, world)
        if not near.any():
            assert [o["recv"][k] for o in outs] == [lo[g + 1] - lo[g] for g in range(world)]
