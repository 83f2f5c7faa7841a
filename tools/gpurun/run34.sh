mkdir -p gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r34.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > gpurun_out/launch_bench.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 2 --launch-count 1 -f -o gpurun_out/k1_async_c2 python tools/k1_once.py > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:route_compact_fast --launch-skip 0 --launch-count 1 -f -o gpurun_out/k3_fast_c2 python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls gpurun_out/*.ncu-rep | tail -3
