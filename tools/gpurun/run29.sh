for v in ldg async; do
  echo "== $v"; HS_CONF_IMPL=$v timeout 300 python tools/breakdown.py 2>&1 | tail -1
done
for c in c1 c4 c5; do for v in ldg async; do
  HS_CONF_IMPL=$v timeout 300 python bench.py --config $c --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$c $v', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1))"
done; done
