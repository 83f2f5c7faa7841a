timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for mode in cluster fused split; do HS_CALIB_MODE=$mode python tools/breakdown.py --reps 30 > gpurun_out/bd13_$mode.json 2>&1; echo $mode; cat gpurun_out/bd13_$mode.json; done
HS_NO_PDL=1 python tools/breakdown.py --reps 30 > gpurun_out/bd13_nopdl.json 2>&1; echo nopdl; cat gpurun_out/bd13_nopdl.json
for p in 0 1; do HS_NO_PDL=$p python bench.py --steps 300 --warmup 5 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b13_$p.json 2> gpurun_out/b13_$p.err; tail -2 gpurun_out/b13_$p.err; python -c "
import json; d=json.load(open('gpurun_out/b13_$p.json')); print('nopdl=$p', round(d['value']/1e6,1), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2))"; done
python bench.py --config c4 --steps 30 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/b13_c4.json 2> gpurun_out/b13_c4.err; tail -2 gpurun_out/b13_c4.err; python -c "
import json; d=json.load(open('gpurun_out/b13_c4.json')); print('c4', round(d['value']/1e6,3), round(d['ms_per_step'],4), round(d['roofline']['achieved']), round(d['roofline']['avg_launch_ms']*1000,2), d['reach'])"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:conf_cta -s 5 -c 1 -o gpurun_out/cta13 python bench.py --config c4 --steps 3 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu13.log 2>&1; tail -1 gpurun_out/ncu13.log
