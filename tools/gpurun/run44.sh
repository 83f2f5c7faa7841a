timeout 900 python bench.py 2>gpurun_out/bench44.err | tail -1 > gpurun_out/bench44.json
cat gpurun_out/bench44.json
for c in c1 c3 c4 c5; do timeout 600 python bench.py --config $c --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench44_$c.json; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r44.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
