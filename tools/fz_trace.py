"""Where the time of a fused cascade step goes (experiment build with
HS_FZ_TRACE, globaltimer stamps): for each C2 routing stage launched alone
(dense layout, live counts from a fixed tensor), the time from the first CTA's
start to the last tile's completion, to the sequencer's last prefix, and to the
last owner's scatter, next to the launch's CUDA-event time.

  python tools/build_variants.py fztrace
  HS_LIBHS=build/exp/libhs_fztrace.so python tools/fz_trace.py
"""
from __future__ import annotations

import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import bench
    import paper_2505_12566_b200 as hs

    dev = torch.device("cuda", 0)
    fam = bench.family("c2")
    route, val, labels, payload = bench.build_inputs(fam, 0, dev)
    router = bench.make_router(fam, dev, None)
    os.environ["HS_FUSE"] = "0"
    route, _ = bench.dense_stage_logits(fam, router, route, val, labels, payload, 0, dev)
    os.environ["HS_FUSE"] = "1"
    K = fam.K
    fixed_n = router.cascade.counts[:, 1].clone()
    thr = router.cal["t"]
    L = hs.lib()
    L.hs_fz_trace.argtypes = [ctypes.POINTER(ctypes.c_ulonglong), ctypes.c_int]
    buf = (ctypes.c_ulonglong * 8)()
    ws = hs.workspace(L.hs_cascade_step_workspace(fam.n, 1), dev)
    out = {}
    for k in range(1, K):
        s = router.stages[k]
        rows = []
        for rep in range(12):
            L.hs_fz_trace(buf, 1)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            hs.cascade_step(k, K, route[k], thr[k:k + 1], n=fam.n, n_classes=s.n_classes,
                            temperature=s.temperature, d_n=fixed_n[k - 1:k], ws=ws)
            e1.record()
            torch.cuda.synchronize()
            L.hs_fz_trace(buf, 0)
            t0 = buf[0]
            rows.append({"event_us": round(e0.elapsed_time(e1) * 1e3, 2),
                         "last_tile_us": (buf[1] - t0) / 1e3, "seq_done_us": (buf[2] - t0) / 1e3,
                         "last_scatter_us": (buf[3] - t0) / 1e3, "warps": int(buf[4]),
                         "last_chunk_end_us": (buf[5] - t0) / 1e3, "seq_probes": int(buf[6])})
        rows = rows[2:]
        med = {key: sorted(r[key] for r in rows)[len(rows) // 2] for key in rows[0]}
        out[f"stage_{k + 1}"] = {"rows": int(fixed_n[k - 1]), **med}
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
