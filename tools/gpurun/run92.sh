timeout 600 python -m pytest tests/test_gpu_split.py -x -q 2>&1 | tail -15 > gpurun_out/pytest92.txt
