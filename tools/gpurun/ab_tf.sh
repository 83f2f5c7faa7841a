tag=${1:-x}
timeout 900 python -m pytest tests/test_gpu_temperature.py -q > gpurun_out/${tag}_tf_tests.txt 2>&1
for r in 1 2; do
  timeout 300 python bench.py --config c2t --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_tf_new_$r.txt 2>&1
  HS_LIBHS=build/exp/libhs_tffp64.so timeout 300 python bench.py --config c2t --steps 50 --no-cpu-baseline --e2e-steps 0 > gpurun_out/${tag}_tf_old_$r.txt 2>&1
done
