"""In-graph cost of the parts of the bench step, dense layout (the timed one):
CUDA graphs of variants of the C2 step, median of replays, no events between
kernels (PDL overlap intact):

  full        calibration + K routing stages (hs_cascade_step: K1 then K3)
  conf_only   the same K1 launches with the live counts taken from a fixed
              device tensor (no compaction): the floor a fused K1+K3 can reach
  k1_stage_k  routing stage k's K1 alone (one launch per graph node)
  steps_fixed hs_cascade_step of every stage, live counts from a fixed tensor
  val_calib   validation K1 + calibration only

  python tools/stage_cost.py [--config c2] [--reps 200]
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
    from paper_2505_12566_b200 import _abi

    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--only", default="", help="comma-separated variant names")
    ap.add_argument("--verbose", action="store_true")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    fam = bench.family(args.config)
    route, val, labels, payload = bench.build_inputs(fam, 0, dev)
    router = bench.make_router(fam, dev, None)
    # set-up (which requests reach which model) on the two-launch step, so a
    # timing-only experiment build of the fused step cannot change it
    fuse_env = os.environ.get("HS_FUSE")
    os.environ["HS_FUSE"] = "0"
    route, _ = bench.dense_stage_logits(fam, router, route, val, labels, payload, 0, dev)
    if fuse_env is None:
        del os.environ["HS_FUSE"]
    else:
        os.environ["HS_FUSE"] = fuse_env
    K = fam.K
    c = router.cascade
    fixed_n = c.counts[:, 1].clone()          # deferred count of every stage (identical every step)
    ws = [hs.workspace(hs.lib().hs_cascade_step_workspace(fam.n, 1), dev) for _ in range(K)]
    thr = router.cal["t"]

    def conf_only(k, overlap=False):
        s = router.stages[k]
        x = route[k]
        _abi.call("hs_cascade_confidence", k, K, hs._p(x), hs._dtype_code(x), fam.n, 1, int(s.n_classes),
                  int(x.stride(0)), None, hs._p(fixed_n[k - 1:k]) if k else None, float(s.temperature),
                  hs._kind(s.kind), hs._reduce(s.reduce), 0.0, hs._p(thr[k:k + 1]), None, hs._p(ws[k]),
                  ws[k].numel(), hs._p(router.status), 0, hs.HS_STEP_OVERLAP_PREVIOUS if overlap else 0,
                  torch.cuda.current_stream().cuda_stream)

    variants = {
        "full": lambda: (router.calibrate(val, labels), router.route(route, n=fam.n, by_id=False,
                                                                     overlap_first=True)),
        "full_no_overlap": lambda: (router.calibrate(val, labels), router.route(route, n=fam.n, by_id=False)),
        "val_calib": lambda: router.calibrate(val, labels),
        "routing_only": lambda: router.route(route, n=fam.n, by_id=False),
        "conf_only": lambda: (router.calibrate(val, labels), [conf_only(k, k == 0) for k in range(K)]),
        "conf_only_routing": lambda: [conf_only(k) for k in range(K)],
    }
    for k in range(K):
        variants[f"k1_stage_{k + 1}"] = (lambda kk: (lambda: conf_only(kk)))(k)

    # hs_cascade_step of every stage with the live counts from a fixed tensor
    # (each stage independent of the previous one's compaction output)
    outs = [None] * K

    def step_fixed(k):
        s_ = router.stages[k]
        outs[k] = hs.cascade_step(k, K, route[k], thr[k:k + 1], n=fam.n, n_classes=s_.n_classes,
                                  temperature=s_.temperature, kind=s_.kind, reduce=s_.reduce,
                                  d_n=fixed_n[k - 1:k] if k else None, out=outs[k], ws=ws[k],
                                  status=router.status)

    variants["steps_fixed"] = lambda: [step_fixed(k) for k in range(K)]
    for k in range(K):
        variants[f"step_fixed_{k + 1}"] = (lambda kk: (lambda: step_fixed(kk)))(k)

    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    torch.cuda.synchronize()
    res = {}
    only = [x for x in args.only.split(",") if x]
    for name, fn in variants.items():
        if only and name not in only:
            continue
        if args.verbose:
            print(f"[stage_cost] {name}", file=sys.stderr, flush=True)
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
        ts = []
        for _ in range(max(1, args.reps // 10)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(s):
                e0.record(s)
                g.replay()
                e1.record(s)
            s.synchronize()
            ts.append(e0.elapsed_time(e1) * 1e3 / 10)
        ts.sort()
        res[name] = round(ts[len(ts) // 2], 2)
    res["_reach"] = [fam.n] + [int(x) for x in fixed_n[:-1].tolist()]
    res["_how"] = ("tools/stage_cost.py: CUDA graphs of 10 back-to-back copies of each variant, "
                   "median per-copy time in us over the replays, dense layout, 1 B200")
    print(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()
