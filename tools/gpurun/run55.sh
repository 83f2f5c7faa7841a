timeout 1500 python -m pytest tests -m gpu -x -q 2>&1 | tail -3 > gpurun_out/pytest55.txt
timeout 600 python bench.py --config c2t --steps 30 2>gpurun_out/b55.err | tail -1 > gpurun_out/bench55_c2t.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:temp_fit --launch-skip 3 --launch-count 1 -f -o gpurun_out/tf_c2t_final python bench.py --config c2t --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tf_launches.csv python bench.py --config c2t --steps 2 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-graph > /dev/null 2>&1
