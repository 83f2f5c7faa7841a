timeout 600 ncu --set full --import-source on --clock-control none -k regex:temp_fit --launch-skip 3 --launch-count 1 -f -o gpurun_out/tf_c2t_v3 python bench.py --config c2t --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 python bench.py --config c2t --steps 30 2>/dev/null | tail -1 > gpurun_out/bench90_c2t.json
