"""Build A/B experiment variants of libhs.so into build/exp/ (not the product)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_12566_b200 import _build  # noqa: E402

VARIANTS = {
    "ridxall": ["HS_AB_K1_RIDX_ALWAYS"],              # K1a: one instantiation for dense and gathered rows
    "tfsub8": ["HS_TF_SUB_STRIDE=8"],                 # temperature fit: warm start on every 8th row
    "tfsub4": ["HS_TF_SUB_STRIDE=4"],                 # ... every 4th row
    "tffp64": ["HS_AB_TF_FP64_ROW"],                  # temperature fit: per-row moments in fp64 (round 1)
    "noticket": ["HS_AB_NO_TICKET"],                  # K3 tiles by blockIdx (round 1)
    "linargmax": ["HS_AB_LINEAR_ARGMAX"],             # K1a argmax: one compare per vector (round 1)
    "ctrace": ["HS_CALIB_TRACE"],        # globaltimer trace of the calibration kernels
    "noargmax": ["HS_EXP_NOARGMAX"],     # upper bounds: K1 without the argmax ...
    "noexp": ["HS_EXP_NOEXP"],           # ... or without the exponential pass
    "tf768": ["HS_TF_THREADS=768"],      # temperature fit: 24 warps/SM, 85 registers
    "tf1024": ["HS_TF_THREADS=1024"],    # temperature fit: 32 warps/SM, 64 registers
    "topk8": ["HS_TOPK_U=8"],            # Top-K confidence: 8 vectors per lane per chunk
    "topknocand": ["HS_EXP_TOPK_NOCAND"],  # Top-K timing bound without candidate handling
    "topkm2": ["HS_TOPK_MERGE_AT=2"],    # Top-K: merge when 2K candidates are buffered
    "topkm4": ["HS_TOPK_MERGE_AT=4"],    # ... 4K
    "topkm8": ["HS_TOPK_MERGE_AT=8"],
    "topkm4s40": ["HS_TOPK_MERGE_AT=4", "HS_TOPK_SLACK=40"],   # + 40 more buffered slots per lane
    "topkm8s40": ["HS_TOPK_MERGE_AT=8", "HS_TOPK_SLACK=40"],
    "noearly": ["HS_AB_NO_EARLY"],
    "k3acqrel": ["HS_AB_K3_ACQREL"],
    "k1g32": ["HS_AB_K1A_G32"],          # K1a for C <= 1,024 bf16: one row per warp (32 lanes x 4 vectors)     # K3 look-back descriptors with acquire / release       # K1a: no first-row prefetch before the PDL wait
    "fznofin": ["HS_EXP_FZ_NOFINISH"],   # fused step timing bounds: grid barrier, no lists ...
    "fznosync": ["HS_EXP_FZ_NOSYNC"],    # ... no barrier either (K1 + tile counters only)
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        out = os.path.join(ROOT, "build", "exp", f"libhs_{n}.so")
        os.makedirs(os.path.dirname(out), exist_ok=True)
        print(_build.build_libhs(force=True, defines=VARIANTS[n], out=out))
