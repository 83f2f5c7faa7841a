"""Per-phase GPU time of one bench step (CUDA graph with external events
between phases), to see where a step's time goes outside the dominant kernel.

  python tools/breakdown.py [--config c2] [--reps 50]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_2505_12566_b200 as hs

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=50)
    args = ap.parse_args()
    torch.cuda.set_device(0)
    dev = torch.device("cuda", 0)
    fam = bench.family(args.config)
    route, val, labels, payload = bench.build_inputs(fam, 0, dev)
    router = bench.make_router(fam, dev, None)
    K = fam.K
    names = []
    evs = []

    def mark(name):
        e = bench.timing_event()
        e.record()
        names.append(name)
        evs.append(e)

    n = fam.n
    s_conf = [torch.empty(n, dtype=torch.float32, device=dev) for _ in range(K)]
    s_am = [torch.empty(n * fam.L, dtype=torch.int32, device=dev) for _ in range(K)]
    s_ws = [hs.workspace(hs.lib().hs_route_compact_workspace(n), dev) for _ in range(K)]
    s_pos = [torch.empty(n, dtype=torch.int64, device=dev) for _ in range(K)]
    cws = torch.empty(max(16, n * fam.L * 5 + 1024), dtype=torch.uint8, device=dev)

    def step():
        names.clear()
        evs.clear()
        mark("start")
        s0 = router.stages[0]
        hs.confidence_batched(val, [t.temperature for t in router.stages], n=router.n_val,
                              seq_len=s0.seq_len, n_classes=s0.n_classes, kind=s0.kind,
                              reduce=s0.reduce, labels=labels,
                              want_argmax=False, out={"conf": router.vconf_all.view(-1),
                                   "correct": router.vok.view(-1)}, ws=router.conf_ws)
        mark("val_conf(all stages, one launch)")
        hs.calibrate_thresholds(router.vconf, router.vok, log2_bins=router.q, out=router.cal,
                                ws=router.cal_ws)
        mark("calibrate")
        t = router.cal["t"]
        c = router.cascade
        for k, s in enumerate(router.stages):
            prev = c.outs[k - 1] if k else None
            ids = prev["next_ids"] if k else None
            d_n = prev["counts"][1:2] if k else None
            hs.confidence(route[k], n=n, seq_len=s.seq_len, n_classes=s.n_classes,
                          temperature=s.temperature, kind=s.kind, reduce=s.reduce, row_index=ids,
                          d_n=d_n, out={"conf": s_conf[k], "argmax": s_am[k]}, ws=cws)
            mark(f"route_conf[{k}]")
            o = c.outs[k]
            hs.route_compact(s_conf[k], t[k:k + 1], is_last=k == K - 1, n=n, d_n=d_n, ids=ids,
                             pred=s_am[k], pred_len=s.seq_len,
                             out={"acc_ids": o["acc_ids"], "acc_conf": o["acc_conf"],
                                  "acc_pred": o["acc_pred"], "def_ids": o["next_ids"],
                                  "def_pos": s_pos[k],
                                  "counts": o["counts"]}, ws=s_ws[k])
            mark(f"route_compact[{k}]")

    stream = torch.cuda.Stream()
    stream.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    with torch.cuda.stream(stream):
        for _ in range(3):
            step()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        step()
    tot = [0.0] * (len(evs) - 1)
    for _ in range(args.reps):
        g.replay()
        torch.cuda.synchronize()
        for i in range(1, len(evs)):
            tot[i - 1] += evs[i - 1].elapsed_time(evs[i])
    res = {names[i]: round(tot[i - 1] / args.reps * 1000, 2) for i in range(1, len(evs))}
    res["total_us"] = round(sum(tot) / args.reps * 1000, 2)
    res["reach"] = [n] + [int(x) for x in router.cascade.counts[:, 1].tolist()[:-1]]
    print(json.dumps(res))


if __name__ == "__main__":
    main()
