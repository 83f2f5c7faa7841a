timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
python tools/calib_bench.py > gpurun_out/calib14.json 2>&1; cat gpurun_out/calib14.json
python tools/breakdown.py --reps 30 > gpurun_out/bd14.json 2>&1; cat gpurun_out/bd14.json
python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b14_c4.json 2> gpurun_out/b14_c4.err; tail -2 gpurun_out/b14_c4.err; python -c "
import json; d=json.load(open('gpurun_out/b14_c4.json')); print('c4', round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2), d['reach'])"
python bench.py --config c3 --steps 10 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b14_c3.json 2> gpurun_out/b14_c3.err; tail -2 gpurun_out/b14_c3.err; python -c "
import json; d=json.load(open('gpurun_out/b14_c3.json')); print('c3', round(d['value']/1e6,4), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2), d['reach'], d['thresholds'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:calib_select -s 2 -c 1 -o gpurun_out/sel14 python tools/calib_bench.py > gpurun_out/ncu14.log 2>&1; tail -1 gpurun_out/ncu14.log
