timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest68.txt
timeout 1200 python tools/fig8_sweep.py --out gpurun_out/fig8_split.json > gpurun_out/fig8_split.log 2>&1
timeout 600 python bench.py 2>/dev/null | tail -1 > gpurun_out/bench68_c2.json
