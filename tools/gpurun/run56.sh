timeout 900 python -m pytest tests/test_gpu_perf_graph.py -x -q 2>&1 | tail -30 > gpurun_out/pytest56.txt
