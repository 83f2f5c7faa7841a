"""Tune the synthetic winner-margin profile of a family toward the paper's
Table III AP handled fractions: prints the calibrated reach per
stage for candidate margin tuples (oracle only, reduced sizes)."""
import dataclasses
import sys
import os
import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle  # noqa: E402
from workload import synth  # noqa: E402


def reach_of(fam, margin, n=20000, n_val=20000):
    K = fam.K
    vids = np.arange(n_val, dtype=np.int64) + synth.VAL_ID_BASE
    lab = synth.labels_np(fam.seed, vids, 1, fam.C).reshape(-1)
    conf = np.empty((K - 1, n_val))
    ok = np.empty((K, n_val), np.uint8)
    for k in range(K):
        b = synth.logits_np(fam.seed, k, vids, 1, fam.C, fam.thr[k], fam.dtype, margin=margin)
        r = oracle.confidence(b, n_val, 1, fam.C, fam.C, fam.temps[k], kind=fam.kind, labels=lab)
        ok[k] = r["correct"]
        if k < K - 1:
            conf[k] = r["conf"]
    cal = oracle.calibrate(conf, ok, fam.log2_bins)
    ids = np.arange(n, dtype=np.int64)
    cs = np.stack([oracle.confidence(synth.logits_np(fam.seed, k, ids, 1, fam.C, fam.thr[k],
                                                     fam.dtype, margin=margin), n, 1, fam.C, fam.C, fam.temps[k],
                                     kind=fam.kind)["conf"] for k in range(K)])
    st = oracle.cascade(cs, np.asarray(cal["t"], np.float64))
    reach = [int((st >= k).sum()) for k in range(K)]
    return cal, reach, ok.mean(1)


if __name__ == "__main__":
    fam = synth.FAMILIES[sys.argv[1] if len(sys.argv) > 1 else "c2"]
    for m in eval(sys.argv[2]):
        cal, reach, acc = reach_of(fam, tuple(m))
        print(m, "t", np.round(cal["t"], 3).tolist(), "reach", [round(r / reach[0], 3) for r in reach],
              "sum", round(sum(reach) / reach[0], 3), "acc", np.round(acc, 3).tolist(), flush=True)
