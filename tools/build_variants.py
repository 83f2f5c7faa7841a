"""Build A/B experiment variants of libhs.so into build/exp/ (not the product)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_12566_b200 import _build  # noqa: E402

VARIANTS = {
    "lb2": ["HS_WARP_MINB=2"],          # G=8 NV=16 capped at 128 regs (16 warps/SM)
    "g16": ["HS_G16"],                  # G=16 NV=8 (~100 regs, 16 warps/SM)
    "g16lb2": ["HS_G16", "HS_WARP_MINB=2"],
    "ctrace": ["HS_CALIB_TRACE"],
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        out = os.path.join(ROOT, "build", "exp", f"libhs_{n}.so")
        print(_build.build_libhs(force=True, defines=VARIANTS[n], out=out))
