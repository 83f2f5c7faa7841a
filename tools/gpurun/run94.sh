timeout 600 python -m pytest tests/test_gpu_comm.py -x -q 2>&1 | tail -25 > gpurun_out/pytest94.txt
