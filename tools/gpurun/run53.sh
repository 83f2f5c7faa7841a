export HS_LIBHS=build/exp/libhs_tf768.so
timeout 600 python bench.py --config c2t --steps 30 --no-cpu-baseline --e2e-steps 0 2>>gpurun_out/b53.err | tail -1 > gpurun_out/bench53_c2t_tf768.json
