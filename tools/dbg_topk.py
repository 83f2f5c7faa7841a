import numpy as np, torch, sys
sys.path.insert(0, '/root/repo')
import paper_2505_12566_b200 as hs, oracle
sys.path.insert(0, '/root/repo/tests')
from test_gpu_parity import _topk_rows, _bf16_bits, to_dev_bits, host_bits
for C in (2, 7, 129):
  for dtype in ("bf16", "fp32"):
    rng = np.random.default_rng(C)
    for mode in ("normal", "ties", "ascending", "descending", "masked", "tiny"):
        x32 = _topk_rows(rng, 8, C, mode)
        bits = _bf16_bits(x32) if dtype == "bf16" else x32
        x = to_dev_bits(bits, dtype, (C + 7) // 8 * 8)
        for K in (1, 2, 10, 32):
            for T, kind in ((1.0, 0), (0.05, 1), (20.0, 2)):
                r = hs.confidence(x, n=8, n_classes=C, temperature=T, kind=kind, top_k=K)
                torch.cuda.synchronize()
                ref = oracle.confidence(host_bits(x), 8, 1, C, x.stride(0), T, kind=kind, top_k=K)
                g = r["conf"].cpu().numpy(); o = ref["conf"]
                ok = np.allclose(g, o, rtol=1e-5, equal_nan=True)
                if not ok:
                    print("FAIL", C, dtype, mode, K, T, kind, g[:4], o[:4])
print("done")
