timeout 900 python -m pytest tests/test_gpu_temperature.py -x -q 2>&1 | tail -5 > gpurun_out/pytest54.txt
for v in base tf768 tfnopf; do
  unset HS_LIBHS HS_TF_G32
  if [ $v = tf768 ]; then export HS_LIBHS=build/exp/libhs_tf768.so; fi
  if [ $v = tfnopf ]; then export HS_LIBHS=build/exp/libhs_tfnopf.so; fi
  timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>>gpurun_out/b54.err | tail -1 > gpurun_out/bench54_c2t_$v.json
done
