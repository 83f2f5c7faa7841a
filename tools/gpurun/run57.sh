timeout 600 python bench.py --config c2g --steps 30 2>gpurun_out/b57.err | tail -1 > gpurun_out/bench57_c2g.json
tail -3 gpurun_out/b57.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:replay_kernel --launch-skip 3 --launch-count 1 -f -o gpurun_out/replay_c2g python bench.py --config c2g --steps 1 --warmup 3 --no-graph --no-cpu-baseline > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/graph_launches.csv python bench.py --config c2g --steps 2 --warmup 3 --no-cpu-baseline --no-graph > /dev/null 2>&1
