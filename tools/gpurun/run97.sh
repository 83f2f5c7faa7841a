timeout 600 python -m pytest tests/test_gpu_forward.py -x -q 2>&1 | tail -5 > gpurun_out/pytest97.txt
