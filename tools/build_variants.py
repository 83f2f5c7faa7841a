"""Build A/B experiment variants of libhs.so into build/exp/ (not the product)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2505_12566_b200 import _build  # noqa: E402

VARIANTS = {
    "ppcopy": ["HS_PP_COPY"],
    "g8": ["HS_G8"],
    "g8pp": ["HS_G8", "HS_PP_COPY"],
    "tma": [],          # same build; selected at run time with HS_CONF_IMPL=tma
}

if __name__ == "__main__":
    names = sys.argv[1:] or list(VARIANTS)
    for n in names:
        out = os.path.join(ROOT, "build", "exp", f"libhs_{n}.so")
        print(_build.build_libhs(force=True, defines=VARIANTS[n], out=out))
