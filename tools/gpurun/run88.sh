timeout 900 python -m pytest tests/test_gpu_temperature.py tests/test_gpu_perf_graph.py -x -q 2>&1 | tail -15 > gpurun_out/pytest88.txt
timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench88_c2t.json
