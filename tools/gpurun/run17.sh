set -x
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
python bench.py > gpurun_out/b17.json 2> gpurun_out/b17.err; tail -2 gpurun_out/b17.err; cat gpurun_out/b17.json
python bench.py --placement balanced --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b17_bal.json 2> gpurun_out/b17_bal.err; tail -3 gpurun_out/b17_bal.err; cat gpurun_out/b17_bal.json
timeout 300 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/ref17.json 2>&1; cat gpurun_out/ref17.json
for c in c1 c4 c3 c5; do python bench.py --config $c --steps 20 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b17_$c.json 2> gpurun_out/b17_$c.err; tail -2 gpurun_out/b17_$c.err; python -c "
import json; d=json.load(open('gpurun_out/b17_$c.json')); print('$c', d['value'], d['ms_per_step'], d['roofline']['achieved'], d['roofline']['frac'], d['reach'], d['thresholds'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches17.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conf_warp -s 19 -c 1 -o gpurun_out/k1_17 python bench.py --steps 4 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:route_compact -s 10 -c 1 -o gpurun_out/rc17 python bench.py --steps 4 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:calib_fused -s 3 -c 1 -o gpurun_out/cal17 python bench.py --steps 4 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conf_cta -s 4 -c 1 -o gpurun_out/cta17 python bench.py --config c4 --steps 3 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
ls gpurun_out/*17*
