timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
for rep in 1 2; do for v in base lb2 g16 g16lb2; do L=""; if [ $v != base ]; then L=$PWD/build/exp/libhs_$v.so; fi; HS_LIBHS=$L python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab3_$v.json 2> gpurun_out/ab3_$v.err; python -c "
import json; d=json.load(open('gpurun_out/ab3_$v.json')); print('$v', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2))" 2>&1 | tail -1; done; done
python tools/breakdown.py --reps 30 > gpurun_out/bd18.json 2>&1; cat gpurun_out/bd18.json
python tools/calib_bench.py > gpurun_out/calib18.json 2>&1; cat gpurun_out/calib18.json | tr '\n' ' '
