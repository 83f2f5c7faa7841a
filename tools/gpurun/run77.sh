timeout 600 python bench.py --steps 50 2>/dev/null | tail -1 > gpurun_out/bench77_c2.json
