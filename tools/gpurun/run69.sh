timeout 1200 python -m pytest tests/test_gpu_split.py tests/test_gpu_parity.py -x -q 2>&1 | tail -3 > gpurun_out/pytest69.txt
timeout 1200 python tools/fig8_sweep.py --out gpurun_out/fig8_split2.json > gpurun_out/fig8_split2.log 2>&1
