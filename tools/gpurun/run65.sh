timeout 900 python -m pytest tests/test_gpu_temperature.py -x -q 2>&1 | tail -3 > gpurun_out/pytest65.txt
run() { timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>/dev/null | tail -1 > gpurun_out/bench65_$1.json; }
run cpa512
HS_LIBHS=build/exp/libhs_tf768.so run cpa768
HS_TF_G32=1 run cpa512_g32
