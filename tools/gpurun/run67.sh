timeout 1200 python -m pytest tests/test_gpu_split.py -x -q 2>&1 | tail -25 > gpurun_out/pytest67.txt
