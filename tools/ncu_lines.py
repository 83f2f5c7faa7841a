"""Per-source-line dynamic instruction counts of one kernel from an ncu capture.

  python tools/ncu_lines.py <report.ncu-rep> <kernel-substring> [--per N] [--top 40]

ncu's SASS page gives "Instructions Executed" per SASS address; the line table
comes from `nvdisasm -g` of the in-tree build (compiled with -lineinfo), so the
capture must come from the same build.  --per divides the counts (e.g. by the
number of warp-iterations) for a per-iteration view.
"""
from __future__ import annotations

import collections
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def sass_counts(rep: str):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    hdr = rows[1]
    ie = hdr.index("Instructions Executed")
    base = int(rows[2][0], 16)
    return [(int(r[0], 16) - base, int(r[ie])) for r in rows[2:] if len(r) > ie and r[ie].isdigit()]


def line_table(kernel: str):
    so = os.path.join(ROOT, "paper_2505_12566_b200", "libhs.so")
    tmp = tempfile.mkdtemp()
    subprocess.run(["cuobjdump", "-xelf", "all", so], cwd=tmp, capture_output=True)
    amap = {}
    for cub in glob.glob(os.path.join(tmp, "*.cubin")):
        text = subprocess.run(["nvdisasm", "-g", cub], capture_output=True, text=True).stdout
        lines = text.splitlines()
        starts = [i for i, l in enumerate(lines) if l.startswith(".text.") and kernel in l]
        if not starts:
            continue
        cur = None
        for l in lines[starts[0] + 1:]:
            if l.startswith(".text.") or l.startswith("\t.section"):
                break
            m = re.search(r'//## File "([^"]+)", line (\d+)', l)
            if m:
                cur = (os.path.basename(m.group(1)), int(m.group(2)))
                continue
            m = re.match(r"\s+/\*([0-9a-f]{4,5})\*/", l)
            if m:
                amap[int(m.group(1), 16)] = cur
        return amap
    raise SystemExit(f"kernel {kernel} not found in {so}")


def main():
    rep, kernel = sys.argv[1], sys.argv[2]
    per = float(sys.argv[sys.argv.index("--per") + 1]) if "--per" in sys.argv else 1.0
    top = int(sys.argv[sys.argv.index("--top") + 1]) if "--top" in sys.argv else 40
    amap = line_table(kernel)
    by = collections.Counter()
    tot = 0
    for off, n in sass_counts(rep):
        by[amap.get(off)] += n
        tot += n
    src = {}
    for k in by:
        if k and k[0] not in src:
            p = glob.glob(os.path.join(ROOT, "paper_2505_12566_b200", "csrc", k[0]))
            src[k[0]] = open(p[0]).read().splitlines() if p else []
    print(f"total {tot / per:.1f} instructions per unit ({tot} warp instructions)")
    for k, v in by.most_common(top):
        text = src.get(k[0], [])[k[1] - 1].strip()[:80] if k and src.get(k[0]) else ""
        print(f"{v / per:8.1f} {100 * v / tot:5.1f}%  {k[0] if k else '?'}:{k[1] if k else ''}  {text}")


if __name__ == "__main__":
    main()
