"""Fig. 8 analogue (SURVEY 8(d) "Fig.-8 sweep", E10): routing latency vs the size
of the prediction vector and the number of cascade models.

The paper measures its CPU router at ~100 ms per 1 MB prediction vector and
<= 1 ms at 50 KB (Fig. 8).  Here: one hs.Cascade route of a batch
through K models with every non-last threshold at +inf (defer all: every
request visits every model, the worst case), captured in a CUDA graph and
replayed; latency = median CUDA-event time per replay.  Prediction vectors are
fp32 (1 KB = 256 classes ... 1 MB = 262,144 classes); values are random (they
do not change the work: one pass over every logit per visit).

  python tools/fig8_sweep.py [--out gpurun_out/fig8.json] [--reps 30]
"""
from __future__ import annotations

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

SIZES_KB = [1, 4, 16, 64, 256, 1024]
KS = [1, 2, 3, 4, 5]
BATCHES = [1, 64, 1024, 8192]
MAX_BYTES = 8 << 30            # logits per (size, batch) point


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(ROOT, "gpurun_out", "fig8.json"))
    ap.add_argument("--reps", type=int, default=30)
    args = ap.parse_args()
    import torch
    import paper_2505_12566_b200 as hs
    dev = torch.device("cuda:0")
    torch.cuda.set_device(dev)
    rows = []
    for kb in SIZES_KB:
        C = kb * 1024 // 4
        for batch in BATCHES:
            if batch * C * 4 > MAX_BYTES:
                continue
            x = torch.randn(batch, C, device=dev, dtype=torch.float32)
            for K in KS:
                casc = hs.Cascade(batch, [hs.StageSpec(C, 1.0) for _ in range(K)], dev)
                thr = torch.tensor([float("inf")] * (K - 1) + [0.0], dtype=torch.float32, device=dev)
                logits = [x] * K
                s = torch.cuda.Stream(device=dev)
                s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
                with torch.cuda.stream(s):
                    for _ in range(3):
                        casc.route(logits, thr)
                torch.cuda.synchronize()
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=s):
                    casc.route(logits, thr)
                g.replay()
                torch.cuda.synchronize()
                assert int(casc.counts[K - 1, 0].item()) == batch   # everything reached m_K
                ts = []
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                for _ in range(args.reps):
                    with torch.cuda.stream(s):
                        e0.record(s)
                        g.replay()
                        e1.record(s)
                    s.synchronize()
                    ts.append(e0.elapsed_time(e1))
                ts.sort()
                ms = ts[len(ts) // 2]
                nbytes = K * batch * C * 4
                rows.append({"pred_kb": kb, "classes": C, "batch": batch, "K": K,
                             "latency_us": ms * 1e3, "p10_us": ts[len(ts) // 10] * 1e3,
                             "p90_us": ts[(9 * len(ts)) // 10] * 1e3,
                             "us_per_vector_visit": ms * 1e3 / (K * batch),
                             "logits_GBps": nbytes / (ms / 1e3) / 1e9})
                print(json.dumps(rows[-1]), flush=True)
                del casc, g
            del x
            torch.cuda.empty_cache()
    os.makedirs(os.path.dirname(args.out), exist_ok=True)
    json.dump({"rows": rows, "note": __doc__}, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
