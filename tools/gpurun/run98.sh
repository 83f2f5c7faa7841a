timeout 900 python -m pytest tests/test_gpu_split.py tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest98.txt
timeout 300 python - > gpurun_out/lat98.txt 2>&1 <<'PY'
import torch, paper_2505_12566_b200 as hs
x = torch.randn(1, 262144, device="cuda")
for use_ws in (False, True):
    ws = torch.empty(hs.lib().hs_confidence_workspace(1, 1), dtype=torch.uint8, device="cuda") if use_ws else torch.empty(16, dtype=torch.uint8, device="cuda")
    for _ in range(5): hs.confidence(x, ws=ws)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50): hs.confidence(x, ws=ws)
    e1.record(); torch.cuda.synchronize()
    print("split" if use_ws else "no-split", e0.elapsed_time(e1) / 50 * 1e3, "us per 1 MB vector")
PY
