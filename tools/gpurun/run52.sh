timeout 900 python -m pytest tests/test_gpu_temperature.py -x -q 2>&1 | tail -5 > gpurun_out/pytest52.txt
for v in 0 1; do
  if [ $v = 1 ]; then export HS_TF_G32=1; fi
  timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>>gpurun_out/b52.err | tail -1 > gpurun_out/bench52_c2t_$v.json
done
