timeout 900 python -m pytest tests/test_gpu_temperature.py -x -q 2>&1 | tail -25 > gpurun_out/pytest50.txt
