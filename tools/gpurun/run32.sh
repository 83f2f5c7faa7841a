for rep in 1 2; do
for v in ldg async; do for co in -1 100; do
  HS_CARVEOUT=$co HS_CONF_IMPL=$v timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v co=$co', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1))"
done; done; done
HS_CARVEOUT=100 HS_CONF_IMPL=async timeout 300 python tools/breakdown.py 2>&1 | tail -1
