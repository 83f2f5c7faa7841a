timeout 900 python bench.py --config c3m --steps 20 --no-cpu-baseline --e2e-steps 0 2>gpurun_out/b91.err | tail -1 > gpurun_out/bench91_c3m.json
tail -2 gpurun_out/b91.err
