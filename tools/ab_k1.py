"""A/B timing of K1 on one box: CUDA-event median of the C2 validation launch
(5 stages x 50,000 rows, batched) and of the stage-1 sweep (262,144 rows), for
the library selected by HS_LIBHS (default: the product build).  Prints one JSON line.

  HS_LIBHS=build/exp/libhs_base.so python tools/ab_k1.py [--reps 30]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2505_12566_b200 as hs
    from workload import synth, gpu_logits, gpu_labels
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--config", default="c2")
    args = ap.parse_args()
    fam = synth.FAMILIES[args.config]
    dt = torch.bfloat16 if fam.dtype == "bf16" else torch.float32
    nv, n = 50000, 262144
    xs = []
    for k in range(fam.K):
        x = torch.empty(nv, fam.C, dtype=dt, device="cuda")
        gpu_logits(x, fam, k, n=nv, id_base=synth.VAL_ID_BASE)
        xs.append(x)
    lab = torch.empty(nv, dtype=torch.int32, device="cuda")
    gpu_labels(lab, fam, id_base=synth.VAL_ID_BASE, n=nv)
    big = torch.empty(n, fam.C, dtype=dt, device="cuda")
    gpu_logits(big, fam, 0, n=n)
    out_b = {}
    out_s = {}
    ws = torch.zeros(16, dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")

    def timed(fn):
        ts = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for i in range(args.reps + 3):
            flush.zero_()
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            if i >= 3:
                ts.append(e0.elapsed_time(e1))
        ts.sort()
        return ts[len(ts) // 2]

    tb = timed(lambda: out_b.update(hs.confidence_batched(xs, fam.temps, n=nv, labels=lab, out=out_b or None)))
    ts = timed(lambda: out_s.update(hs.confidence(big, temperature=fam.temps[0], out=out_s or None, ws=ws)))
    vb = fam.K * nv * (fam.C * 2 + 13)
    sb = n * (fam.C * 2 + 8)
    print(json.dumps({"lib": os.environ.get("HS_LIBHS", "product"), "val_ms": tb, "val_GBps": vb / tb / 1e6,
                      "stage1_ms": ts, "stage1_GBps": sb / ts / 1e6, "build": hs.build_info()}))


if __name__ == "__main__":
    main()
