"""Summarise ncu captures for profiles/ (run here, on the CPU box).

  python tools/ncu_summary.py full  <report.ncu-rep> [--bytes N]   # one --set full capture
  python tools/ncu_summary.py launches <launches.csv> [--step N]   # gpu__time_duration list
  python tools/ncu_summary.py traffic <report.ncu-rep> <config> <out.json>

`full` prints the headline metrics (duration, DRAM bytes and throughput, issue,
pipe utilisation, stall reasons) and the dynamic SASS opcode mix; `launches`
prints every launch of one step with its share of the step.
"""
from __future__ import annotations

import collections
import csv
import io
import os
import subprocess
import sys

HEAD = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__cycles_elapsed.avg.per_second", "launch__grid_size", "launch__block_size",
    "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
    "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum",
]


def _ncu(args):
    return subprocess.run(["ncu"] + args, capture_output=True, text=True).stdout


def full(path: str, algo_bytes: float | None = None):
    raw = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    name = vals[hdr.index("Kernel Name")] if "Kernel Name" in hdr else "?"
    print(f"kernel: {name}")
    d = {}
    for h, u, v in zip(hdr, units, vals):
        if h in HEAD or ("stall" in h and "ratio" in h and h.startswith("smsp__average_warps_issue")):
            d[h] = (v, u)
    for h in HEAD:
        if h in d:
            print(f"  {h:62s} {d[h][0]:>16s} {d[h][1]}")
    dur = float(d["gpu__time_duration.sum"][0]) * (1e-3 if d["gpu__time_duration.sum"][1] == "ns" else 1.0)
    rd = float(d["dram__bytes_read.sum"][0])
    wr = float(d.get("dram__bytes_write.sum", ("0", ""))[0])
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd *= scale.get(d["dram__bytes_read.sum"][1], 1)
    wr *= scale.get(d.get("dram__bytes_write.sum", ("0", "byte"))[1], 1)
    print(f"  traffic (dram read+write) bytes/launch: {rd + wr:.0f}")
    print(f"  dram GB/s under ncu (cold, serialised): {(rd + wr) / (dur * 1e-6) / 1e9:.0f}")
    if algo_bytes:
        print(f"  algorithmic bytes/launch: {algo_bytes:.0f}  (traffic/algorithmic = {(rd + wr) / algo_bytes:.3f})")
    print("  stall reasons (warps per issue):")
    st = sorted(((float(v[0]), h) for h, v in d.items() if "stall" in h), reverse=True)
    for v, h in st[:8]:
        print(f"    {h.replace('smsp__average_warps_issue_stalled_', '').replace('_per_issue_active.ratio', ''):28s} {v:.3f}")
    src = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "source", "--csv", "--print-source", "sass"]))))
    h = src[1]
    ins, col = h.index("Instructions Executed"), h.index("Source")
    cnt, tot = collections.Counter(), 0
    for row in src[2:]:
        try:
            n = int(row[ins])
        except (ValueError, IndexError):
            continue
        toks = row[col].split()
        if not toks:
            continue
        op = toks[1] if toks[0].startswith("@") and len(toks) > 1 else toks[0]
        cnt[op.split(".")[0]] += n
        tot += n
    print(f"  dynamic SASS mix ({tot} warp instructions):")
    for op, n in cnt.most_common(16):
        print(f"    {op:10s} {n:12d} {100 * n / tot:5.1f}%")


def launches(path: str, step: int | None = None):
    rows = list(csv.reader(open(path)))
    hi = [i for i, r in enumerate(rows) if "Kernel Name" in r][0]
    h = rows[hi]
    ki, vi, ii, mi = h.index("Kernel Name"), h.index("Metric Value"), h.index("ID"), h.index("Metric Name")
    seq = [(int(r[ii]), r[ki].split("(")[0], float(r[vi].replace(",", "")))
           for r in rows[hi + 1:] if r[mi] == "gpu__time_duration.sum"]
    print(f"{len(seq)} launches")
    by = collections.defaultdict(float)
    for _, k, v in seq:
        by[k] += v
    tot = sum(by.values())
    for k, v in sorted(by.items(), key=lambda x: -x[1]):
        print(f"  {100 * v / tot:5.1f}%  {v / 1e3:10.1f} us  {k}")


def traffic(path: str, config: str, out: str):
    """Write the DRAM bytes of one `--set full` capture for bench.py's roofline."""
    import json
    raw = list(csv.reader(io.StringIO(_ncu(["-i", path, "--page", "raw", "--csv"]))))
    hdr, units, vals = raw[0], raw[1], raw[2]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    tot = 0.0
    for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
        i = hdr.index(key)
        tot += float(vals[i]) * scale.get(units[i], 1)
    rec = {"config": config, "kernel": vals[hdr.index("Kernel Name")],
           "dram_bytes_per_launch": int(round(tot)), "source": os.path.basename(path),
           "capture": "ncu --set full --clock-control none (one launch)"}
    json.dump(rec, open(out, "w"), indent=1)
    print(rec)


if __name__ == "__main__":
    mode, path = sys.argv[1], sys.argv[2]
    if mode == "full":
        b = float(sys.argv[sys.argv.index("--bytes") + 1]) if "--bytes" in sys.argv else None
        full(path, b)
    elif mode == "traffic":       # traffic <report> <config> <out.json>
        traffic(path, sys.argv[3], sys.argv[4])
    else:
        launches(path)
