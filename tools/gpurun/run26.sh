timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -3
for rep in 1 2; do
for v in default noargmax; do
  if [ $v = default ]; then L=""; else L=$PWD/build/exp/libhs_$v.so; fi
  HS_LIBHS=$L timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$v', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1))"
done; done
