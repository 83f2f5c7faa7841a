"""Time hs_calibrate_thresholds alone (graph-replayed) across modes, K, q, N."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import paper_2505_12566_b200 as hs
    dev = torch.device("cuda", 0)
    g = torch.Generator(device="cpu").manual_seed(0)
    res = {}
    for N in (4096, 50000, 1 << 20):
        for K in (2, 5):
            conf = torch.rand(K - 1, N, generator=g).to(dev)
            ok = (torch.rand(K, N, generator=g) < 0.8).to(torch.uint8).to(dev)
            for q in (4, 12):
                for mode in ("cluster", "fused", "fused_streaming", "split"):
                    if mode == "cluster" and N >= (1 << 20):
                        continue
                    os.environ["HS_CALIB_MODE"] = mode.split("_")[0]
                    if mode == "fused_streaming":
                        os.environ["HS_CALIB_NORESIDENT"] = "1"
                    else:
                        os.environ.pop("HS_CALIB_NORESIDENT", None)
                    out = hs._calib_out(K, dev, None)
                    ws = hs.calibrate_workspace(K, q, dev)
                    s = torch.cuda.Stream()
                    s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
                    with torch.cuda.stream(s):
                        for _ in range(3):
                            hs.calibrate_thresholds(conf, ok, log2_bins=q, out=out, ws=ws)
                    torch.cuda.synchronize()
                    gr = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(gr, stream=s):
                        for _ in range(10):
                            hs.calibrate_thresholds(conf, ok, log2_bins=q, out=out, ws=ws)
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    gr.replay()
                    torch.cuda.synchronize()
                    e0.record()
                    for _ in range(5):
                        gr.replay()
                    e1.record()
                    torch.cuda.synchronize()
                    res[f"N={N} K={K} q={q} {mode}"] = round(e0.elapsed_time(e1) / 50 * 1000, 2)
    os.environ.pop("HS_CALIB_MODE", None)
    # an empty kernel pair for reference: hs_route_compact on n = 0 inside a graph
    c = torch.empty(0, device=dev)
    ws = hs.workspace(hs.lib().hs_route_compact_workspace(0), dev)
    out = {}
    o = hs.route_compact(c, 0.5, ws=ws)
    gr = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())   # after the set-up queued so far
    with torch.cuda.graph(gr, stream=s):
        for _ in range(20):
            hs.route_compact(c, 0.5, ws=ws, out=o)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    gr.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(5):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    res["route_compact n=0 (per launch)"] = round(e0.elapsed_time(e1) / 100 * 1000, 2)
    print(json.dumps(res, indent=0))


if __name__ == "__main__":
    main()
