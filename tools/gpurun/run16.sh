timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python tools/calib_bench.py > gpurun_out/calib16.json 2>&1; cat gpurun_out/calib16.json | tr '\n' ' '; echo
python tools/breakdown.py --reps 30 > gpurun_out/bd16.json 2>&1; cat gpurun_out/bd16.json
python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b16.json 2> gpurun_out/b16.err; tail -2 gpurun_out/b16.err; python -c "
import json; d=json.load(open('gpurun_out/b16.json')); print(round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2))"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conf_warp -s 0 -c 1 -o gpurun_out/val16 python bench.py --steps 3 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu16.log 2>&1; tail -1 gpurun_out/ncu16.log
