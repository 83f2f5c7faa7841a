"""In-graph marginal cost of each part of the bench step (no events between
kernels, so PDL overlap is intact): time CUDA graphs of growing prefixes of the
step -- validation K1, + calibration, + routing stage 1 (overlapped), + each
later stage -- and print the increments.

  python tools/ablate.py [--config c2] [--reps 100] [--no-overlap]
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
    ap.add_argument("--reps", type=int, default=100)
    ap.add_argument("--no-overlap", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    fam = bench.family(args.config)
    route, val, labels, payload = bench.build_inputs(fam, 0, dev)
    router = bench.make_router(fam, dev, None)
    K = fam.K
    c = router.cascade

    def prefix(upto):
        # upto: 0 = val K1, 1 = + calibration, 2 + k = + routing stages 0..k
        def run():
            router.calibrate(val, labels) if upto >= 1 else None
            if upto == 0:
                s0 = router.stages[0]
                hs.confidence_batched(val, [t.temperature for t in router.stages], n=router.n_val,
                                      seq_len=s0.seq_len, n_classes=s0.n_classes, kind=s0.kind,
                                      reduce=s0.reduce, labels=labels,
                                      want_argmax=False, out={"conf": router.vconf_all.view(-1),
                                           "correct": router.vok.view(-1)}, ws=router.conf_ws)
            thr = router.cal["t"]
            for k in range(0, max(0, upto - 1)):
                s = router.stages[k]
                prev = c.outs[k - 1] if k else None
                hs.cascade_step(k, K, route[k], thr[k:k + 1], n=fam.n, seq_len=s.seq_len,
                                n_classes=s.n_classes, temperature=s.temperature, kind=s.kind,
                                reduce=s.reduce, row_index=prev["next_ids"] if k else None,
                                d_n=prev["counts"][1:2] if k else None,
                                ids=prev["next_ids"] if k else None,
                                payload=prev.get("next_payload") if k else payload,
                                payload_row_bytes=c.P, out=c.outs[k], ws=c.ws, status=router.status,
                                overlap_previous=(k == 0 and not args.no_overlap))
        return run

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    res = {}
    prev_t = 0.0
    names = ["val K1", "+ calibration"] + [f"+ stage {k + 1}" for k in range(K)]
    for upto in range(len(names)):
        fn = prefix(upto)
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=s):
            for _ in range(10):
                fn()
        g.replay()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(args.reps // 10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) * 1e3 / (args.reps // 10 * 10)
        res[names[upto]] = {"total_us": round(t, 2), "delta_us": round(t - prev_t, 2)}
        prev_t = t
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
