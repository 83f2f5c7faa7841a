timeout 600 python bench.py --native-comm --steps 20 --no-cpu-baseline --e2e-steps 0 2>gpurun_out/b95.err | tail -1 > gpurun_out/bench95_native.json
tail -2 gpurun_out/b95.err
