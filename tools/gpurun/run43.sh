timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_async --launch-skip 20 --launch-count 1 -f -o gpurun_out/k1_stage2 python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:route_compact_fast --launch-skip 15 --launch-count 2 -f -o gpurun_out/k3_stage12 python bench.py --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls -la gpurun_out/k1_stage2.ncu-rep gpurun_out/k3_stage12.ncu-rep
