timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for rep in 1 2; do for o in "" "--no-overlap"; do
  timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1), d['gpu_launches_per_step'])"
done; done
