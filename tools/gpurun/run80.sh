timeout 900 python -m pytest tests/test_gpu_perf_graph.py -x -q -k router 2>&1 | tail -25 > gpurun_out/pytest80.txt
