timeout 900 python -m pytest tests/test_gpu_perf_graph.py -x -q 2>&1 | tail -30 > gpurun_out/pytest58.txt
timeout 600 python bench.py --config c2g --steps 30 --no-cpu-baseline 2>gpurun_out/b58.err | tail -1 > gpurun_out/bench58_c2g.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay_hist --launch-skip 3 --launch-count 1 -f -o gpurun_out/replay_hist_c2g python bench.py --config c2g --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/graph_launches2.csv python bench.py --config c2g --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
