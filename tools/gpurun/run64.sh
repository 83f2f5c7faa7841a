timeout 900 python -m pytest tests/test_gpu_perf_graph.py -x -q 2>&1 | tail -3 > gpurun_out/pytest64.txt
timeout 600 python bench.py --config c2g --steps 30 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench64_c2g.json
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/graph_launches3.csv python bench.py --config c2g --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
