"""Build the native libraries in-tree with nvcc (sm_100a only).

* paper_2505_12566_b200/libhs.so  -- the product: kernels + C-ABI (include/hs.h)
* workload/libhs_synth.so         -- the synthetic-input generator (not product)
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import shutil
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
LIBHS = os.path.join(PKG, "libhs.so")
SYNTH_SRC = os.path.join(ROOT, "workload", "csrc", "synth.cu")
LIBSYNTH = os.path.join(ROOT, "workload", "libhs_synth.so")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
NVCC_FLAGS = ARCH + ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                     "-Xcompiler", "-O2", "-diag-suppress", "550"]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target: str, sources) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(s) > t for s in sources)


def _run(cmd):
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("build failed: " + " ".join(cmd) + "\n" + r.stdout + r.stderr)
    return r


def build_libhs(force: bool = False, verbose: bool = False, defines=(), out: str | None = None) -> str:
    """Build libhs.so; `defines` + `out` build an experiment variant (A/B only)."""
    target = out or LIBHS
    cus = sorted(glob.glob(os.path.join(CSRC, "*.cu")))
    deps = cus + glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) + \
        [os.path.join(ROOT, "include", "hs.h")]
    if not force and not _stale(target, deps):
        return target
    objdir = os.path.join(ROOT, "build", os.path.basename(target)[:-3])
    os.makedirs(objdir, exist_ok=True)
    nv = nvcc()
    objs = []
    cmds = []
    for cu in cus:
        o = os.path.join(objdir, os.path.basename(cu)[:-3] + ".o")
        objs.append(o)
        cmds.append([nv] + NVCC_FLAGS + [f"-D{d}" for d in defines] + ["-c", cu, "-o", o])
    with cf.ThreadPoolExecutor(max_workers=min(8, len(cmds))) as ex:
        for r in ex.map(_run, cmds):
            if verbose:
                print(r.stderr)
    tmp = target + f".tmp{os.getpid()}"
    _run([nv] + ARCH + ["-shared", "-o", tmp] + objs)
    os.replace(tmp, target)
    return target


def build_synth(force: bool = False) -> str:
    if not force and not _stale(LIBSYNTH, [SYNTH_SRC]):
        return LIBSYNTH
    tmp = LIBSYNTH + f".tmp{os.getpid()}"
    _run([nvcc()] + NVCC_FLAGS + ["-shared", SYNTH_SRC, "-o", tmp])
    os.replace(tmp, LIBSYNTH)
    return LIBSYNTH


def build_all(force: bool = False, verbose: bool = False):
    return build_libhs(force, verbose), build_synth(force)


if __name__ == "__main__":
    import sys
    print(build_all(force="--force" in sys.argv, verbose="-v" in sys.argv))
