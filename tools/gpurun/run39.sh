timeout 600 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | grep -E "^E |passed|failed" | head -30
for rep in 1 2; do for o in "" "--no-overlap"; do
  timeout 300 python bench.py --e2e-steps 0 --no-cpu-baseline $o 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$o', round(d['roofline']['achieved']), round(d['roofline']['frac'],3), round(d['ms_per_step']*1000,1), d['gpu_launches_per_step'])"
done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_ --launch-skip 2 --launch-count 1 -f -o gpurun_out/k1_val_b5 python tools/k1_once.py --rows 50000 --batched 5 > /dev/null 2>&1
