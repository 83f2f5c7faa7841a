"""Run K1 (hs_confidence) on the C2 stage-1 shape a few times -- a target for
`ncu -k regex:conf_ --launch-skip 2 --launch-count 1` captures.

  python tools/k1_once.py [--config c2] [--rows 262144] [--reps 4]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2505_12566_b200 as hs
    from workload import synth, gpu_logits
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--rows", type=int, default=262144)
    ap.add_argument("--reps", type=int, default=4)
    ap.add_argument("--batched", type=int, default=0, help="K stages of --rows each, one launch")
    args = ap.parse_args()
    fam = synth.FAMILIES[args.config]
    dt = torch.bfloat16 if fam.dtype == "bf16" else torch.float32
    if args.batched:
        xs = []
        for k in range(args.batched):
            xk = torch.empty(args.rows * fam.L, fam.C, dtype=dt, device="cuda")
            gpu_logits(xk, fam, k, n=args.rows, id_base=synth.VAL_ID_BASE)
            xs.append(xk)
        lab = torch.randint(0, fam.C, (args.rows * fam.L,), dtype=torch.int32, device="cuda")
        for _ in range(args.reps):
            hs.confidence_batched(xs, fam.temps[:args.batched], n=args.rows, seq_len=fam.L, want_argmax=False,
                                  kind=fam.kind, reduce=fam.reduce, labels=lab)
        torch.cuda.synchronize()
        print("ok")
        return
    x = torch.empty(args.rows * fam.L, fam.C, dtype=dt, device="cuda")
    gpu_logits(x, fam, 0, n=args.rows)
    for _ in range(args.reps):
        hs.confidence(x, n=args.rows, seq_len=fam.L, temperature=fam.temps[0], kind=fam.kind,
                      reduce=fam.reduce)
    torch.cuda.synchronize()
    print("ok")


if __name__ == "__main__":
    main()
