timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
HS_CONF_IMPL=ldg timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "conf or cascade" 2>&1 | tail -2
for rep in 1 2; do
  timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('new', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1))"
done
timeout 300 python tools/breakdown.py 2>&1 | tail -1
