timeout 1200 python tools/fig8_sweep.py --out gpurun_out/fig8.json > gpurun_out/fig8.log 2>&1
tail -3 gpurun_out/fig8.log
