"""Print the stage_cost A/B lines of one gpurun tag (tools/gpurun/fzab.sh)."""
import glob
import json
import sys

tag = sys.argv[1]
for f in sorted(glob.glob(f"gpurun_out/{tag}_sc_*.txt")):
    try:
        d = json.load(open(f))
        print(f.split("_sc_")[1][:-4], {k: v for k, v in d.items() if k.startswith(("step", "k1", "full", "routing"))})
    except Exception as e:
        print(f, e)
