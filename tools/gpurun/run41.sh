timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "^E |passed|failed" | head -30
for rep in 1 2; do
  timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1))"
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_r41.csv python bench.py --steps 2 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
