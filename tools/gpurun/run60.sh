timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -5 > gpurun_out/pytest60.txt
for v in stream cta; do
  unset HS_CONF_IMPL
  if [ $v = cta ]; then export HS_CONF_IMPL=cta; fi
  for c in c3 c4; do timeout 900 python bench.py --config $c --e2e-steps 0 --steps 20 --no-cpu-baseline 2>/dev/null | tail -1 > gpurun_out/bench60_${c}_$v.json; done
done
unset HS_CONF_IMPL
timeout 600 ncu --set full --import-source on --clock-control none -k regex:conf_stream --launch-skip 3 --launch-count 1 -f -o gpurun_out/k1d_c3 python bench.py --config c3 --steps 1 --warmup 3 --no-graph --no-cpu-baseline --e2e-steps 0 > /dev/null 2>&1
